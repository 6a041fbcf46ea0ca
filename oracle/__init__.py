"""CPU oracle for arXiv 1210.1878's hot path (ctypes binding of liboracle.so).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product path
(paper_1210_1878_b200) never imports it, and the two share no code: the C sources here
(assemble.c, ainv.c, pcg.c) are written from PAPER.md and DESIGN.md only.

Functions (all fp64; unknown vectors are ocean points in natural order):
  assemble(problem)               -> Assembled  (A as CSR, Eq. 9-10)
  Assembled.apply(x)              -> A x
  Assembled.anchor_check()        -> -1 or the first unanchored unknown
  ainv(asm, tau, ...)             -> Ainv  (Zhat, pivots, scale)
  fsai(asm, q)                    -> Ainv  (the paper's banded FSAI of T)
  pcg(asm, b, ...)                -> PcgResult (Alg. 1, d = s + beta d)
  partition(nj, ni, mask, parts)  -> row bounds
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["assemble.c", "ainv.c", "fsai.c", "pcg.c"]

ERR = {0: "OK", 1: "ARG", 2: "NOT_SPD", 3: "BREAKDOWN", 6: "NOMEM"}
PRECOND = {"ainv": 0, "jacobi": 1, "none": 2}
MODE = {"plain": 0, "canonical": 1, "chunked": 2}


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C11, -O3 -march=x86-64-v3 -ffp-contract=off, OpenMP; no CUDA)."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES]
    hdrs = [os.path.join(_HERE, h) for h in ("oracle.h", "oracle_internal.h")]
    if not force and os.path.exists(_LIB_PATH):
        t = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(s) <= t for s in srcs + hdrs):
            return _LIB_PATH
    # -O3 for x86-64-v3 (AVX2: every host of this pool); -ffp-contract=off and no fast-math keep
    # each sum and product one IEEE operation in the written order; OpenMP only in the CHUNKED
    # mode's row loops and chunk partials (results independent of the thread count)
    cmd = ["gcc", "-std=c11", "-O3", "-march=x86-64-v3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-Wall", "-Wno-unused-function", "-o", _LIB_PATH] + srcs + ["-lm"]
    subprocess.run(cmd, check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        vp = C.c_void_p
        L.orc_assemble.argtypes = [I32, I32, I32, vp, vp, vp, vp, C.POINTER(P)]
        L.orc_assemble.restype = C.c_int
        L.orc_problem_free.argtypes = [P]
        L.orc_n.argtypes = [P]; L.orc_n.restype = I64
        L.orc_nnz.argtypes = [P]; L.orc_nnz.restype = I64
        L.orc_csr.argtypes = [P, vp, vp, vp]
        L.orc_grid_index.argtypes = [P, vp]
        L.orc_diag.argtypes = [P, vp]
        L.orc_apply.argtypes = [P, vp, vp]
        L.orc_anchor_check.argtypes = [P]; L.orc_anchor_check.restype = I64
        L.orc_partition.argtypes = [I32, I32, vp, I32, vp]
        L.orc_ainv_build.argtypes = [P, D, I32, I32, I32, C.POINTER(P), C.POINTER(I64)]
        L.orc_ainv_build.restype = C.c_int
        L.orc_ainv_build_fill.argtypes = [P, D, I32, I32, I32, I32, C.POINTER(P), C.POINTER(I64)]
        L.orc_ainv_build_fill.restype = C.c_int
        L.orc_fsai_build.argtypes = [P, I32, C.POINTER(P), C.POINTER(I64)]
        L.orc_fsai_build.restype = C.c_int
        L.orc_ainv_free.argtypes = [P]
        L.orc_ainv_nnz.argtypes = [P]; L.orc_ainv_nnz.restype = I64
        L.orc_ainv_export.argtypes = [P, vp, vp, vp, vp, vp, vp]
        L.orc_ainv_apply.argtypes = [P, vp, vp]
        L.orc_apply_canonical.argtypes = [P, vp, vp]
        L.orc_ainv_apply_canonical.argtypes = [P, vp, vp]
        L.orc_dot_canonical.argtypes = [P, vp, vp, vp]
        L.orc_dot_canonical.restype = D
        L.orc_pcg.argtypes = [P, P, vp, vp, vp, D, I32, vp, vp, vp]
        L.orc_pcg.restype = C.c_int
        L.orc_pcg_cg.argtypes = [P, P, vp, vp, vp, D, I32, vp, vp, vp]
        L.orc_pcg_cg.restype = C.c_int
        L.orc_pcg_pipe.argtypes = [P, P, vp, vp, vp, D, I32, vp, vp, vp]
        L.orc_pcg_pipe.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle {ERR.get(code, code)} {msg}")
        self.code = ERR.get(code, code)


class _PcgOpts(C.Structure):
    _fields_ = [("precond", C.c_int32), ("mode", C.c_int32), ("pitch", C.c_int32),
                ("block", C.c_int32), ("parts", C.c_int32), ("rows", C.c_int32)]


class _PcgReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("rel_residual", C.c_double), ("true_rel_residual", C.c_double),
                ("failed_index", C.c_int64)]


class Assembled:
    """A (Eq. 10 negated, masked, E-W periodic) as CSR over the ocean unknowns."""

    def __init__(self, ni, nj, cE, cN, mask, periodic=True, sigma=None):
        L = lib()
        self.ni, self.nj = int(ni), int(nj)
        self._cE = np.ascontiguousarray(cE, dtype=np.float64)
        self._cN = np.ascontiguousarray(cN, dtype=np.float64)
        self._mask = np.ascontiguousarray(mask, dtype=np.uint8)
        self._sigma = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
        h = C.c_void_p()
        rc = L.orc_assemble(self.ni, self.nj, 1 if periodic else 0, _ptr(self._cE), _ptr(self._cN),
                            _ptr(self._sigma), _ptr(self._mask), C.byref(h))
        if rc != 0:
            raise OracleError(rc, "assemble")
        self._h = h
        self.n = int(L.orc_n(h))
        self.nnz = int(L.orc_nnz(h))
        self.grid_index = np.empty(self.n, dtype=np.int64)
        L.orc_grid_index(h, _ptr(self.grid_index))

    @classmethod
    def from_problem(cls, p):
        return cls(p.ni, p.nj, p.cE, p.cN, p.mask, p.periodic, p.sigma)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.orc_problem_free(h)
            self._h = None

    def csr(self):
        rp = np.empty(self.n + 1, dtype=np.int64)
        col = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz, dtype=np.float64)
        lib().orc_csr(self._h, _ptr(rp), _ptr(col), _ptr(val))
        return rp, col, val

    def dense(self):
        rp, col, val = self.csr()
        A = np.zeros((self.n, self.n))
        for p in range(self.n):
            A[p, col[rp[p]:rp[p + 1]]] = val[rp[p]:rp[p + 1]]
        return A

    def diag(self):
        d = np.empty(self.n)
        lib().orc_diag(self._h, _ptr(d))
        return d

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        lib().orc_apply(self._h, _ptr(x), _ptr(y))
        return y

    def apply_canonical(self, x):
        """y = A x in the GPU's documented order."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        lib().orc_apply_canonical(self._h, _ptr(x), _ptr(y))
        return y

    def dot_canonical(self, a, b, pitch, block=256, parts=1, rows=1):
        o = _PcgOpts(0, 1, int(pitch), int(block), int(parts), int(rows))
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return float(lib().orc_dot_canonical(self._h, C.byref(o), _ptr(a), _ptr(b)))

    def anchor_check(self) -> int:
        return int(lib().orc_anchor_check(self._h))

    # grid <-> unknown helpers (layout only)
    def to_grid(self, v):
        g = np.zeros(self.ni * self.nj)
        g[self.grid_index] = v
        return g.reshape(self.nj, self.ni)

    def from_grid(self, g):
        return np.ascontiguousarray(np.asarray(g, dtype=np.float64).reshape(-1)[self.grid_index])


def assemble(p) -> Assembled:
    return Assembled.from_problem(p)


@dataclasses.dataclass
class Ainv:
    colptr: np.ndarray
    row: np.ndarray
    zhat: np.ndarray
    z: np.ndarray
    pivots: np.ndarray
    scale: np.ndarray
    handle: object = None

    @property
    def n(self):
        return len(self.pivots)

    @property
    def nnz_offdiag(self):
        return len(self.row) - self.n

    def zhat_dense(self):
        Z = np.zeros((self.n, self.n))
        for j in range(self.n):
            Z[self.row[self.colptr[j]:self.colptr[j + 1]], j] = self.zhat[self.colptr[j]:self.colptr[j + 1]]
        return Z

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        s = np.empty(self.n)
        lib().orc_ainv_apply(self.handle._h, _ptr(r), _ptr(s))
        return s

    def apply_canonical(self, r):
        """s = Z D^-1 Z^T r in the GPU's documented order."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        s = np.empty(self.n)
        lib().orc_ainv_apply_canonical(self.handle._h, _ptr(r), _ptr(s))
        return s


class _AinvHandle:
    def __init__(self, h):
        self._h = h

    def __del__(self):
        if self._h is not None and _lib is not None:
            _lib.orc_ainv_free(self._h)
            self._h = None


def ainv(A: Assembled, tau: float, method: str = "sparse", parts: int = 1, halo: int = 0, fill: int = 0) -> Ainv:
    """AINV(A, tau) (P_B1); fill = m > 0 adds P_B2's count rule (m entries per column incl. the
    diagonal, reading R26)."""
    L = lib()
    h = C.c_void_p()
    fail = C.c_int64(-1)
    rc = L.orc_ainv_build_fill(A._h, float(tau), int(fill), 1 if method == "dense" else 0, int(parts), int(halo),
                               C.byref(h), C.byref(fail))
    if rc != 0:
        e = OracleError(rc, f"ainv failed at column {fail.value}")
        e.index = fail.value
        raise e
    nnz = int(L.orc_ainv_nnz(h))
    n = A.n
    cp = np.empty(n + 1, dtype=np.int64)
    row = np.empty(nnz, dtype=np.int64)
    zh = np.empty(nnz)
    z = np.empty(nnz)
    pv = np.empty(n)
    sc = np.empty(n)
    L.orc_ainv_export(h, _ptr(cp), _ptr(row), _ptr(zh), _ptr(z), _ptr(pv), _ptr(sc))
    return Ainv(cp, row, zh, z, pv, sc, _AinvHandle(h))


def fsai(A: Assembled, q: int) -> Ainv:
    """The paper's banded FSAI of T = band(A, 1) (Eq. 19), bandwidth q, as an
    AINV-form factor: unit-diagonal zhat, pivots u_kk^2, scale 1 (P = Zhat D^-1 Zhat^t)."""
    L = lib()
    h = C.c_void_p()
    fail = C.c_int64(-1)
    rc = L.orc_fsai_build(A._h, int(q), C.byref(h), C.byref(fail))
    if rc != 0:
        e = OracleError(rc, f"fsai failed at unknown {fail.value}")
        e.index = fail.value
        raise e
    nnz = int(L.orc_ainv_nnz(h))
    n = A.n
    cp = np.empty(n + 1, dtype=np.int64)
    row = np.empty(nnz, dtype=np.int64)
    zh = np.empty(nnz)
    z = np.empty(nnz)
    pv = np.empty(n)
    sc = np.empty(n)
    L.orc_ainv_export(h, _ptr(cp), _ptr(row), _ptr(zh), _ptr(z), _ptr(pv), _ptr(sc))
    return Ainv(cp, row, zh, z, pv, sc, _AinvHandle(h))


@dataclasses.dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    hist: np.ndarray
    rel_residual: float
    true_rel_residual: float
    status: str


def pcg(A: Assembled, b, precond: str = "ainv", M: Ainv | None = None, tol: float = 1e-10,
        maxit: int | None = None, x0=None, mode: str = "plain", pitch: int | None = None,
        block: int = 256, parts: int = 1, rows: int = 1, method: str = "pcg") -> PcgResult:
    """Alg. 1 with d = s + beta d.  Unknown-indexed vectors.
    method = "cg1": Chronopoulos-Gear single-reduction form (NEXT-2, orc_pcg_cg);
    method = "pipe": pipelined PCG, Ghysels-Vanroose Alg. 4 (NEXT-2, orc_pcg_pipe)."""
    L = lib()
    if maxit is None:
        maxit = A.n
    b = np.ascontiguousarray(b, dtype=np.float64)
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    x = np.empty(A.n)
    hist = np.empty(maxit + 1)
    o = _PcgOpts(PRECOND[precond], MODE[mode], int(pitch if pitch else A.ni), int(block), int(parts), int(rows))
    rep = _PcgReport()
    fn = {"pcg": L.orc_pcg, "cg1": L.orc_pcg_cg, "pipe": L.orc_pcg_pipe}[method]
    rc = fn(A._h, None if M is None else M.handle._h, C.byref(o), _ptr(b), _ptr(x0a),
            float(tol), int(maxit), _ptr(x), _ptr(hist), C.byref(rep))
    if rc == 1:
        raise OracleError(rc, "pcg")
    k = rep.iterations
    return PcgResult(x, k, bool(rep.converged), hist[:k + 1].copy(), rep.rel_residual,
                     rep.true_rel_residual, ERR.get(rep.status, str(rep.status)))


def partition(nj: int, ni: int, mask, parts: int) -> np.ndarray:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    rb = np.empty(parts + 1, dtype=np.int32)
    lib().orc_partition(int(nj), int(ni), _ptr(m), int(parts), _ptr(rb))
    return rb
