"""The C-ABI boundary without a GPU: libpcg.so loads, exports every function declared in
include/libpcg.h, and its host setup (validation, partition, anchor check, AINV) agrees
with the oracle bit for bit (the two share no code)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_1210_1878_b200 as pcg
from paper_1210_1878_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "libpcg.h")
INF = float("inf")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:pcg_status|void|const char\*|int64_t)\s+(pcg_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", pcg.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (pcg_\w+)$", out, re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = pcg.lib()
    for n in names:
        assert hasattr(L, n)
    assert set(names) == set(pcg.EXPORTS)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", pcg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_partition_matches_oracle(name):
    p = synth.config(name)
    for P in (1, 2, 3, 4, 8):
        assert np.array_equal(pcg.partition(p.ni, p.nj, p.mask, P), oracle.partition(p.nj, p.ni, p.mask, P))


def _compare(p, tau, parts=0, halo=0):
    A = oracle.assemble(p)
    ref = oracle.ainv(A, tau, parts=max(1, parts), halo=halo)
    pl = pcg.Plan(p.cE, p.cN, p.mask, periodic=p.periodic, tau=tau, sigma=p.sigma, ainv_parts=parts, ainv_halo=halo)
    cp, row, zh, pv, sc = pl.export_zhat()
    assert pl.n_owned == A.n
    assert np.array_equal(cp, ref.colptr)
    assert np.array_equal(row, ref.row)
    assert np.array_equal(zh, ref.zhat)          # bitwise
    assert np.array_equal(pv, ref.pivots)
    assert np.array_equal(sc, ref.scale)
    return pl


@pytest.mark.parametrize("tau", [0.0, 0.05 + 1e-9, 0.1 + 1e-9, 0.2 + 1e-9, INF])
@pytest.mark.parametrize("shape", [(9, 8, 1), (13, 11, 4)])
@pytest.mark.parametrize("periodic", [True, False])
def test_host_ainv_bitwise_equals_oracle_small(tau, shape, periodic):
    p = synth.random_grid(*shape, periodic=periodic, sigma=shape[2] == 4)
    _compare(p, tau)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_host_ainv_bitwise_equals_oracle_configs(name):
    pl = _compare(synth.config(name), 0.1 + 1e-9)
    assert pl.pitch % 32 == 0 and pl.pitch >= synth.config(name).ni


@pytest.mark.parametrize("parts", [2, 3, 8])
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_global_z_is_rank_count_invariant(name, parts):
    """NEXT-3: with every block starting at row 0 (halo >= nj) the partitioned AINV
    is the one-block AINV bit for bit, in the oracle and in the library -- the left-looking column
    j only involves rows and columns < j, so its owner's row range does not
    matter.  A wrong halo clamp or a block that drops southern rows breaks the equality."""
    p = synth.config(name)
    A = oracle.assemble(p)
    one = oracle.ainv(A, 0.1 + 1e-9)
    glob = oracle.ainv(A, 0.1 + 1e-9, parts=parts, halo=p.nj)
    for f in ("colptr", "row", "zhat", "pivots", "scale"):
        assert np.array_equal(getattr(glob, f), getattr(one, f))
    local = oracle.ainv(A, 0.1 + 1e-9, parts=parts, halo=0)   # block-local differs (sanity)
    assert local.row.size != one.row.size or not np.array_equal(local.zhat, one.zhat)
    _compare(p, 0.1 + 1e-9, parts, p.nj)


@pytest.mark.parametrize("parts,halo", [(2, 0), (4, 0), (4, 3), (8, 1)])
def test_host_partitioned_ainv_bitwise_equals_oracle(parts, halo):
    _compare(synth.config("cfg2"), 0.1 + 1e-9, parts, halo)


def test_setup_errors_without_gpu():
    p = synth.random_grid(8, 6, 1)
    cE = p.cE.copy(); cE[2, 3] = np.nan
    with pytest.raises(pcg.PcgError) as e:
        pcg.Plan(cE, p.cN, p.mask)
    assert e.value.code == "ERR_ARG" and "(i=3, j=2)" in str(e.value)
    with pytest.raises(pcg.PcgError) as e:
        pcg.Plan(p.cE[:, :2], p.cN[:, :2], p.mask[:, :2])
    assert e.value.code == "ERR_ARG"
    with pytest.raises(pcg.PcgError) as e:
        pcg.Plan(p.cE, p.cN, p.mask, tau=float("nan"))
    assert e.value.code == "ERR_ARG"
    q = synth.singular_channel(16, 6, 3)
    with pytest.raises(pcg.PcgError) as e:
        pcg.Plan(q.cE, q.cN, q.mask)
    assert e.value.code == "ERR_NOT_SPD" and "anchor" in str(e.value)
    # tau = 0 on a tiny SPD grid works; on the singular grid the anchor check fires first
    pcg.Plan(p.cE, p.cN, p.mask, tau=0.0)


def test_sell_padding_is_small():
    """full-grid SELL-32 rows pad by ~1.15-1.25 at tau = 0.1."""
    p = synth.config("cfg3")
    pl = pcg.Plan(p.cE, p.cN, p.mask, tau=0.1 + 1e-9)
    nnz = pl.nnz
    assert 1.0 < pl.sell_z / nnz < 1.35 and 1.0 < pl.sell_zt / nnz < 1.35


# ---------------------------------------------------------------- NEXT-1: the paper's FSAI
def _fsai_equal(p, q):
    A = oracle.assemble(p)
    M = oracle.fsai(A, q)
    pl = pcg.Plan(p.cE, p.cN, p.mask, periodic=p.periodic, sigma=p.sigma, precond="fsai", fsai_q=q)
    cp, r, z, pv, sc = pl.export_zhat()
    assert np.array_equal(cp, M.colptr) and np.array_equal(r, M.row)
    assert np.array_equal(z, M.zhat) and np.array_equal(pv, M.pivots) and np.array_equal(sc, M.scale)
    return A, M


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
@pytest.mark.parametrize("q", [0, 1, 4, 16])
def test_host_fsai_bitwise_equals_oracle_configs(name, q):
    """The library's banded FSAI of T (csrc/fsai.cpp) equals the oracle's (oracle/fsai.c) bit
    for bit: factor, pivots u_kk^2, unit scale (reading R25)."""
    _fsai_equal(synth.config(name), q)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("periodic", [True, False])
def test_host_fsai_bitwise_literal_band(seed, periodic):
    """Land-heavy random grids: consecutive unknowns are also periodic-wrap or N-S neighbours
    here (T = band(A, 1) taken literally), and sigma > 0 enters the diagonal."""
    p = synth.random_grid(7, 9, seed, land_frac=0.6, periodic=periodic, sigma=True)
    A, M = _fsai_equal(p, 6)
    gi = A.grid_index
    D = A.dense()
    # the factor's couplings are exactly A's entries between consecutive unknowns
    sup = np.array([D[k, k + 1] for k in range(A.n - 1)])
    linked = np.array([(M.row[M.colptr[k + 1]:M.colptr[k + 2]] == k).any() for k in range(A.n - 1)])
    assert np.array_equal(linked, sup != 0)


def test_fsai_setup_errors():
    p = synth.config("cfg1")
    with pytest.raises(pcg.PcgError):
        pcg.Plan(p.cE, p.cN, p.mask, precond="fsai", fsai_q=-1)
    with pytest.raises(pcg.PcgError):
        pcg.Plan(p.cE, p.cN, p.mask, precond="fsai", fsai_q=4, j_begin=0, j_end=16, rank=0, nranks=2)


def test_host_fsai_wrap_coupling():
    """A row whose only ocean points are i = 0 and i = ni-1 on a periodic grid: the two
    consecutive unknowns are coupled through the wrap face, which T = band(A, 1) keeps."""
    ni, nj = 6, 4
    rng = np.random.default_rng(7)
    mask = np.zeros((nj, ni), dtype=np.uint8)
    mask[1, 0] = mask[1, ni - 1] = 1
    mask[2, 1:4] = 1
    cE = rng.uniform(0.5, 2.0, (nj, ni)); cN = rng.uniform(0.5, 2.0, (nj, ni)); cN[nj - 1] = 0.0
    p = synth.Problem("wrap", ni, nj, cE, cN, mask, True, None)
    A, M = _fsai_equal(p, 3)
    D = A.dense()
    assert D[0, 1] == -cE[1, ni - 1]                       # unknowns 0, 1 = (0,1), (5,1)
    assert M.row[M.colptr[1]] == 0 and M.zhat[M.colptr[1]] != 0.0


# ---------------------------------------------------------------- NEXT-4: P_B2 (fixed fill)
def _pb2_equal(p, tau, fill, **kw):
    A = oracle.assemble(p)
    M = oracle.ainv(A, tau, fill=fill, parts=max(1, kw.get("ainv_parts", 0) or 1), halo=kw.get("ainv_halo", 0))
    pl = pcg.Plan(p.cE, p.cN, p.mask, periodic=p.periodic, sigma=p.sigma, tau=tau, ainv_fill=fill, **kw)
    cp, r, z, pv, sc = pl.export_zhat()
    assert np.array_equal(cp, M.colptr) and np.array_equal(r, M.row)
    assert np.array_equal(z, M.zhat) and np.array_equal(pv, M.pivots) and np.array_equal(sc, M.scale)


@pytest.mark.parametrize("name,fill", [("cfg1", 2), ("cfg1", 4), ("cfg2", 3), ("cfg2", 6), ("cfg3", 5)])
def test_host_pb2_bitwise_equals_oracle(name, fill):
    """The library's fixed-fill AINV (csrc/ainv.cpp) equals the oracle's bit for bit, incl. the
    tie rule on cfg1's constant couplings."""
    _pb2_equal(synth.config(name), 0.0, fill)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_host_pb2_with_tau_and_partitions(seed):
    p = synth.random_grid(17, 14, seed, sigma=True, periodic=seed != 2)
    _pb2_equal(p, 0.02 + 1e-9, 4)
    _pb2_equal(p, 0.0, 3, ainv_parts=3, ainv_halo=2)


@pytest.mark.parametrize("name,fill", [("cfg3", 0), ("cfg3", 5), ("cfg4", 0)])
def test_threaded_ainv_equals_one_thread(name, fill):
    """The column wavefront of ainv.cpp (several threads, each column waiting only on the finished
    columns it reads) builds bitwise the single-thread factor, and at cfg3 the oracle's."""
    p = synth.config(name)
    tau = 0.0 if fill else 0.1 + 1e-9
    one = pcg.Plan(p.cE, p.cN, p.mask, tau=tau, ainv_fill=fill, setup_threads=1).export_zhat()
    for th in (3, 8):
        many = pcg.Plan(p.cE, p.cN, p.mask, tau=tau, ainv_fill=fill, setup_threads=th).export_zhat()
        assert all(np.array_equal(a, b) for a, b in zip(one, many))
    if name == "cfg3":
        A = oracle.assemble(p)
        M = oracle.ainv(A, tau, fill=fill)
        cp, row, zh, pv, sc = one
        assert np.array_equal(cp, M.colptr) and np.array_equal(row, M.row) and np.array_equal(zh, M.zhat)
        assert np.array_equal(pv, M.pivots)
