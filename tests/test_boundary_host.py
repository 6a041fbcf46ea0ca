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
