"""paper_1210_1878_b200 -- Python face of libpcg (B200-native fp64 PCG + AINV, arXiv 1210.1878).

Argument marshalling only: every step of the solve runs in libpcg.so's CUDA kernels
(csrc/).  There is NO CPU fallback: if libpcg.so is missing or fails to load, every call
raises.  PyTorch is used for device memory, streams and process groups only.

    from paper_1210_1878_b200 import Solver, synth
    p = synth.config("cfg4")
    S = Solver(p.cE, p.cN, p.mask, tau=0.1)              # pcg_setup
    x, it, hist, rep = S.solve(b, tol=1e-10)             # pcg_solve (torch CUDA tensors)
    S.close()                                            # pcg_free

The C ABI is include/libpcg.h; the names below mirror it (pcg_setup, pcg_solve,
pcg_solve_host, pcg_free, pcg_apply_operator, pcg_partition, ...).
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCG_LIB") or os.path.join(_HERE, "libpcg.so")   # PCG_LIB: tuning variants

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_NOT_SPD", 3: "ERR_BREAKDOWN", 4: "ERR_CUDA", 5: "ERR_COMM", 6: "ERR_NOMEM"}
PRECOND = {"ainv": 0, "jacobi": 1, "none": 2, "fsai": 3}
FLAG_HOST_LOOP = 1
FLAG_COMM_PATH = 2
FLAG_LOCAL_RANKS = 4
FLAG_SINGLE_REDUCTION = 8
FLAG_PIPELINED = 16
FLAG_DEVICE_COMM = 32


class PcgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = STATUS.get(code, str(code))
        super().__init__(f"libpcg {self.code}: {msg}")


class Grid(C.Structure):
    _fields_ = [("ni", C.c_int32), ("nj", C.c_int32), ("periodic_ew", C.c_int32),
                ("j_begin", C.c_int32), ("j_end", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_comm", C.c_void_p), ("device", C.c_int32), ("stream", C.c_void_p)]


class Coeffs(C.Structure):
    _fields_ = [("cE", C.c_void_p), ("cN", C.c_void_p), ("sigma", C.c_void_p), ("mask", C.c_void_p)]


class Opts(C.Structure):
    _fields_ = [("precond", C.c_int32), ("drop_tol", C.c_double), ("flags", C.c_int32),
                ("ainv_parts", C.c_int32), ("ainv_halo", C.c_int32), ("setup_threads", C.c_int32),
                ("fsai_q", C.c_int32), ("ainv_fill", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("rel_residual", C.c_double),
                ("true_rel_residual", C.c_double), ("setup_s", C.c_double), ("solve_s", C.c_double),
                ("bytes_per_iter", C.c_double), ("n_ocean", C.c_int64), ("nnz_z", C.c_int64),
                ("failed_index", C.c_int64), ("driver", C.c_int32), ("kernels_per_iter", C.c_int32)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["driver_name"] = DRIVERS.get(d["driver"], str(d["driver"]))
        return d


DRIVERS = {0: "graph", 1: "loop", 2: "resident", 3: "host_loop", 4: "nccl_graph", 5: "nccl_fallback_host_loop",
           6: "nccl_host_loop", 7: "local_ranks"}


EXPORTS = ["pcg_setup", "pcg_solve", "pcg_solve_host", "pcg_solve_local_ranks", "pcg_free", "pcg_last_error", "pcg_apply_operator",
           "pcg_apply_preconditioner", "pcg_extrapolate", "pcg_partition", "pcg_layout", "pcg_kernel_times", "pcg_device_bytes", "pcg_loop_time",
           "pcg_plan_build", "pcg_plan_free", "pcg_plan_counts", "pcg_plan_export_zhat",
           "pcg_comm_unique_id", "pcg_comm_init_rank", "pcg_comm_destroy", "pcg_devcomm_selftest"]

_lib = None


def lib():
    """Load libpcg.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libpcg.so not found at {LIB_PATH}: build it with "
                          f"`python -m paper_1210_1878_b200.build` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.pcg_setup.argtypes = [C.POINTER(Coeffs), C.POINTER(Grid), C.POINTER(Opts), C.POINTER(vp)]
    L.pcg_solve.argtypes = [vp, vp, vp, d, i32, vp, C.POINTER(i32), vp, i32, C.POINTER(Report)]
    L.pcg_solve_host.argtypes = L.pcg_solve.argtypes
    L.pcg_solve_local_ranks.argtypes = [C.POINTER(vp), i32, vp, vp, d, i32, vp, C.POINTER(i32), vp, i32, C.POINTER(Report)]
    L.pcg_free.argtypes = [vp]; L.pcg_free.restype = None
    L.pcg_last_error.argtypes = [vp]; L.pcg_last_error.restype = C.c_char_p
    L.pcg_apply_operator.argtypes = [vp, vp, vp]
    L.pcg_apply_preconditioner.argtypes = [vp, vp, vp]
    L.pcg_extrapolate.argtypes = [vp, vp, vp, vp]
    L.pcg_partition.argtypes = [i32, i32, vp, i32, vp]
    L.pcg_layout.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
    L.pcg_kernel_times.argtypes = [vp, i32, vp, vp]
    L.pcg_device_bytes.argtypes = [vp]; L.pcg_device_bytes.restype = i64
    L.pcg_loop_time.argtypes = [vp, C.POINTER(d), C.POINTER(i32)]
    L.pcg_plan_build.argtypes = [C.POINTER(Coeffs), C.POINTER(Grid), C.POINTER(Opts), C.POINTER(vp)]
    L.pcg_plan_free.argtypes = [vp]; L.pcg_plan_free.restype = None
    L.pcg_plan_counts.argtypes = [vp, vp]
    L.pcg_plan_export_zhat.argtypes = [vp, vp, vp, vp, vp, vp]
    L.pcg_comm_unique_id.argtypes = [C.c_char_p]
    L.pcg_comm_init_rank.argtypes = [C.c_char_p, i32, i32, i32, C.POINTER(vp)]
    L.pcg_comm_destroy.argtypes = [vp]
    L.pcg_devcomm_selftest.argtypes = [i32, i32, C.c_uint64, vp]
    for f in EXPORTS:
        if f not in ("pcg_free", "pcg_last_error", "pcg_device_bytes", "pcg_plan_free"):
            getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _check(rc, ctx=None, what=""):
    if rc != 0:
        msg = lib().pcg_last_error(ctx)
        raise PcgError(rc, (msg.decode() if msg else "") or what)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def devcomm_selftest(nranks: int, rounds: int, seed: int = 1) -> np.ndarray:
    """pcg_devcomm_selftest: [rounds][nranks][4] rank trees of the device-comm protocol run by
    nranks virtual ranks on the current device."""
    out = np.empty((rounds, nranks, 4))
    _check(lib().pcg_devcomm_selftest(int(nranks), int(rounds), int(seed), _ptr(out)), None, "pcg_devcomm_selftest")
    return out


def partition(ni: int, nj: int, mask, parts: int) -> np.ndarray:
    """Documented row-block split (pcg_partition)."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    rb = np.empty(parts + 1, dtype=np.int32)
    _check(lib().pcg_partition(int(ni), int(nj), _ptr(m), int(parts), _ptr(rb)), None, "pcg_partition")
    return rb


def _host_inputs(cE, cN, mask, sigma):
    cE = np.ascontiguousarray(cE, dtype=np.float64)
    cN = np.ascontiguousarray(cN, dtype=np.float64)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    sigma = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
    return cE, cN, mask, sigma


def _opts(precond, tau, flags, ainv_parts, ainv_halo, setup_threads, fsai_q=4, ainv_fill=0):
    return Opts(PRECOND[precond], float(tau), int(flags), int(ainv_parts), int(ainv_halo), int(setup_threads),
                int(fsai_q), int(ainv_fill))


class Plan:
    """Host-only half of pcg_setup (validation, partition, anchor check, AINV, SELL packing)."""

    def __init__(self, cE, cN, mask, *, periodic=True, tau=0.1, precond="ainv", sigma=None,
                 j_begin=None, j_end=None, rank=0, nranks=1, ainv_parts=0, ainv_halo=0, setup_threads=0, fsai_q=4,
                 ainv_fill=0):
        L = lib()
        cE, cN, mask, sigma = _host_inputs(cE, cN, mask, sigma)
        nj, ni = mask.shape
        self._keep = (cE, cN, mask, sigma)
        co = Coeffs(_ptr(cE), _ptr(cN), _ptr(sigma), _ptr(mask))
        g = Grid(ni, nj, 1 if periodic else 0, 0 if j_begin is None else j_begin, nj if j_end is None else j_end,
                 rank, nranks, None, 0, None)
        o = _opts(precond, tau, 0, ainv_parts, ainv_halo, setup_threads, fsai_q, ainv_fill)
        h = C.c_void_p()
        _check(L.pcg_plan_build(C.byref(co), C.byref(g), C.byref(o), C.byref(h)), None, "pcg_plan_build")
        self._h = h
        cnt = np.empty(6, dtype=np.int64)
        L.pcg_plan_counts(h, _ptr(cnt))
        self.n_owned, self.nnz, self.pitch, self.sell_z, self.sell_zt, self.first_global = (int(v) for v in cnt)

    def export_zhat(self):
        cp = np.empty(self.n_owned + 1, dtype=np.int64)
        row = np.empty(self.nnz, dtype=np.int64)
        zh = np.empty(self.nnz)
        pv = np.empty(self.n_owned)
        sc = np.empty(self.n_owned)
        lib().pcg_plan_export_zhat(self._h, _ptr(cp), _ptr(row), _ptr(zh), _ptr(pv), _ptr(sc))
        return cp, row, zh, pv, sc

    def close(self):
        if getattr(self, "_h", None) is not None:
            lib().pcg_plan_free(self._h)
            self._h = None

    __del__ = close


class Solver:
    """pcg_setup / pcg_solve / pcg_free on one rank.

    cE, cN, mask (and sigma): global [nj][ni] host arrays (numpy).  With a torch process
    group of size > 1, rows are split by `partition` and an NCCL communicator is created
    (uid broadcast over the group); setup and solve are then collective.
    """

    def __init__(self, cE, cN, mask, *, periodic=True, tau=0.1, precond="ainv", sigma=None,
                 group=None, device=None, stream=None, flags=0, ainv_parts=0, ainv_halo=0,
                 setup_threads=0, comm_path=False, fsai_q=4, ainv_fill=0):
        import torch
        import torch.distributed as dist
        L = lib()
        cE, cN, mask, sigma = _host_inputs(cE, cN, mask, sigma)
        nj, ni = mask.shape
        self.ni, self.nj = ni, nj
        self.n_ocean = int(np.count_nonzero(mask))     # N_o: the default maxit (Alg. 1's k <= n)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        torch.cuda.set_device(self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.rank, self.nranks = 0, 1
        self._comm = None
        if group is not None or (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
            if dist.is_initialized():
                self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        if self.nranks > 1 or comm_path:
            uid = C.create_string_buffer(128)
            if self.rank == 0:
                _check(L.pcg_comm_unique_id(uid), None, "pcg_comm_unique_id")
            if self.nranks > 1:
                obj = [bytes(uid.raw) if self.rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                uid = C.create_string_buffer(obj[0], 128)
            comm = C.c_void_p()
            _check(L.pcg_comm_init_rank(uid, self.nranks, self.rank, self.device.index, C.byref(comm)),
                   None, "pcg_comm_init_rank")
            self._comm = comm
            if comm_path:
                flags |= FLAG_COMM_PATH
        rb = partition(ni, nj, mask, self.nranks)
        self.j_begin, self.j_end = int(rb[self.rank]), int(rb[self.rank + 1])
        self.rows = self.j_end - self.j_begin
        co = Coeffs(_ptr(cE), _ptr(cN), _ptr(sigma), _ptr(mask))
        g = Grid(ni, nj, 1 if periodic else 0, self.j_begin, self.j_end, self.rank, self.nranks,
                 self._comm, self.device.index, self.stream.cuda_stream)
        o = _opts(precond, tau, flags, ainv_parts, ainv_halo, setup_threads, fsai_q, ainv_fill)
        h = C.c_void_p()
        _check(L.pcg_setup(C.byref(co), C.byref(g), C.byref(o), C.byref(h)), None, "pcg_setup")
        self._h = h
        p, b, r = C.c_int32(), C.c_int32(), C.c_int32()
        L.pcg_layout(h, C.byref(p), C.byref(b), C.byref(r))
        self.pitch, self.block, self.tile_rows = p.value, b.value, r.value
        self.precond = precond

    # -- solve -----------------------------------------------------------------------------
    def solve(self, b, x0=None, tol=1e-10, maxit=None, x=None, hist_cap=None):
        """b, x0, x: torch CUDA float64 [rows][ni] (this rank's rows).  Returns
        (x, iterations, hist (numpy), report dict)."""
        import torch
        if maxit is None:
            maxit = self.n_ocean
        assert b.is_cuda and b.dtype == torch.float64 and b.is_contiguous() and tuple(b.shape) == (self.rows, self.ni)
        if x is None:
            x = torch.empty_like(b)
        assert x.is_cuda and x.dtype == torch.float64 and x.is_contiguous() and x.shape == b.shape
        if x0 is not None:
            assert x0.is_cuda and x0.dtype == torch.float64 and x0.is_contiguous() and x0.shape == b.shape
        cap = int(hist_cap if hist_cap is not None else min(maxit + 1, 1 << 22))
        hist = np.empty(max(cap, 1))
        it = C.c_int32()
        rep = Report()
        rc = lib().pcg_solve(self._h, _ptr(b), _ptr(x0), float(tol), int(maxit), _ptr(x), C.byref(it),
                             _ptr(hist), cap, C.byref(rep))
        _check(rc, self._h, "pcg_solve")
        k = it.value
        return x, k, hist[:min(k + 1, cap)].copy(), rep.as_dict()

    def solve_host(self, b, x0=None, tol=1e-10, maxit=None, out=None, hist_cap=None):
        """Same with host numpy (or pinned torch CPU) buffers; the H2D/D2H copies happen inside
        pcg_solve_host."""
        if maxit is None:
            maxit = self.n_ocean
        shape = (self.rows, self.ni)
        b = np.ascontiguousarray(b, dtype=np.float64)
        assert b.shape == shape, f"b must be {shape}"
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
            assert x0.shape == shape, f"x0 must be {shape}"
        if out is None:
            out = np.empty(shape)
        assert isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == shape and out.flags.c_contiguous, \
            f"out must be a C-contiguous float64 {shape} array"
        cap = int(hist_cap if hist_cap is not None else min(maxit + 1, 1 << 22))
        hist = np.empty(max(cap, 1))
        it = C.c_int32()
        rep = Report()
        rc = lib().pcg_solve_host(self._h, _ptr(b), _ptr(x0), float(tol), int(maxit), _ptr(out), C.byref(it),
                                  _ptr(hist), cap, C.byref(rep))
        _check(rc, self._h, "pcg_solve_host")
        k = it.value
        return out, k, hist[:min(k + 1, cap)].copy(), rep.as_dict()

    def apply_operator(self, x, y=None):
        import torch
        y = torch.empty_like(x) if y is None else y
        _check(lib().pcg_apply_operator(self._h, _ptr(x), _ptr(y)), self._h, "pcg_apply_operator")
        return y

    def apply_preconditioner(self, r, s=None):
        import torch
        s = torch.empty_like(r) if s is None else s
        _check(lib().pcg_apply_preconditioner(self._h, _ptr(r), _ptr(s)), self._h, "pcg_apply_preconditioner")
        return s

    def extrapolate(self, x_t, x_tm1, x0=None):
        """NEMO's first guess 2 x_t - x_tm1 (pcg_extrapolate; torch CUDA float64 [rows][ni])."""
        import torch
        x0 = torch.empty_like(x_t) if x0 is None else x0
        _check(lib().pcg_extrapolate(self._h, _ptr(x_t), _ptr(x_tm1), _ptr(x0)), self._h, "pcg_extrapolate")
        return x0

    def kernel_times(self, n_iter=50):
        ms = np.zeros(4)
        by = np.zeros(3)
        _check(lib().pcg_kernel_times(self._h, int(n_iter), _ptr(ms), _ptr(by)), self._h, "pcg_kernel_times")
        return ms, by

    def loop_time(self):
        """(ms, iterations) of the resident-strip loop kernel in the last solve; ms = -1 when the
        solve used another driver (pcg_loop_time)."""
        ms, it = C.c_double(-1.0), C.c_int32(0)
        _check(lib().pcg_loop_time(self._h, C.byref(ms), C.byref(it)), self._h, "pcg_loop_time")
        return ms.value, it.value

    @property
    def device_bytes(self):
        return int(lib().pcg_device_bytes(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None:
            lib().pcg_free(self._h)
            self._h = None
        if getattr(self, "_comm", None) is not None:
            lib().pcg_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalRanks:
    """One-GPU emulation of an n-rank row-block run (pcg_solve_local_ranks): n contexts, one per
    row block of `partition`, stepped phase by phase with device-copy exchanges.  Exercises the
    multi-rank device code path (halo rows, rank sums, rank-ordered tree) without n GPUs."""

    def __init__(self, cE, cN, mask, nranks, *, periodic=True, tau=0.1, precond="ainv", sigma=None, device=None,
                 setup_threads=0, ainv_halo=0, ainv_fill=0, flags=0):
        import torch
        L = lib()
        cE, cN, mask, sigma = _host_inputs(cE, cN, mask, sigma)
        nj, ni = mask.shape
        self.ni, self.nj, self.n = ni, nj, int(nranks)
        self.n_ocean = int(np.count_nonzero(mask))
        dev = torch.cuda.current_device() if device is None else int(device)
        stream = torch.cuda.current_stream(dev)
        self.rb = partition(ni, nj, mask, self.n)
        co = Coeffs(_ptr(cE), _ptr(cN), _ptr(sigma), _ptr(mask))
        self._h = []
        for r in range(self.n):
            g = Grid(ni, nj, 1 if periodic else 0, int(self.rb[r]), int(self.rb[r + 1]), r, self.n, None, dev,
                     stream.cuda_stream)
            o = _opts(precond, tau, FLAG_LOCAL_RANKS | int(flags), 0, int(ainv_halo), setup_threads, 4, ainv_fill)
            h = C.c_void_p()
            rc = L.pcg_setup(C.byref(co), C.byref(g), C.byref(o), C.byref(h))
            if rc != 0:
                self.close()
                _check(rc, None, "pcg_setup")
            self._h.append(h)
        p, b, t = C.c_int32(), C.c_int32(), C.c_int32()
        L.pcg_layout(self._h[0], C.byref(p), C.byref(b), C.byref(t))
        self.pitch, self.block = p.value, b.value

    def solve(self, b, x0=None, tol=1e-10, maxit=None, x=None, hist_cap=None):
        import torch
        if maxit is None:
            maxit = self.n_ocean
        assert b.is_cuda and b.dtype == torch.float64 and b.is_contiguous() and tuple(b.shape) == (self.nj, self.ni)
        x = torch.empty_like(b) if x is None else x
        cap = int(hist_cap if hist_cap is not None else min(maxit + 1, 1 << 22))
        hist = np.empty(max(cap, 1))
        it = C.c_int32()
        rep = Report()
        arr = (C.c_void_p * self.n)(*[h.value for h in self._h])
        rc = lib().pcg_solve_local_ranks(arr, self.n, _ptr(b), _ptr(x0), float(tol), int(maxit), _ptr(x), C.byref(it),
                                         _ptr(hist), cap, C.byref(rep))
        _check(rc, self._h[0], "pcg_solve_local_ranks")
        k = it.value
        return x, k, hist[:min(k + 1, cap)].copy(), rep.as_dict()

    def close(self):
        for h in getattr(self, "_h", []):
            if h is not None:
                lib().pcg_free(h)
        self._h = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
