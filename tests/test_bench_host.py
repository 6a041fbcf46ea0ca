"""bench.py's host-side accounting without a GPU: the operator's entry count against the oracle's
assembled CSR matrix, and the SPEC S:387 flop model against its own worked example."""
import dataclasses
import os
import sys

import numpy as np
import pytest

import oracle
from paper_1210_1878_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("p", [synth.config("cfg1"), synth.config("cfg2"),
                               synth.random_grid(17, 11, 3, periodic=False),
                               synth.random_grid(16, 9, 4, periodic=True)], ids=lambda p: p.name)
def test_nnz_operator_matches_assembled_matrix(p):
    assert bench.nnz_operator(p) == oracle.assemble(p).nnz


def test_flop_model_isolated_points_is_12n():
    # S:387 example: identity A (nnz = n), no preconditioner, one iteration -> 12 n.  A checkerboard
    # mask on a non-periodic grid leaves no two ocean points adjacent, so A is diagonal.
    p = synth.random_grid(12, 10, 5, land_frac=0.0, periodic=False)
    jj, ii = np.mgrid[0:p.nj, 0:p.ni]
    mask = (((ii + jj) % 2) == 0).astype(np.uint8)
    mask[0, :] = 0
    mask[-1, :] = 0
    q = dataclasses.replace(p, mask=mask)
    n = int(mask.sum())
    assert bench.nnz_operator(q) == n == oracle.assemble(q).nnz
    assert bench.flop_model(q, "none", 0, 1) == 12 * n
    assert bench.flop_model(q, "jacobi", 0, 3) == 3 * 13 * n


def test_flop_model_factored_counts_both_factors():
    p = synth.config("cfg1")
    n, nnzA = p.n_ocean, bench.nnz_operator(p)
    M = oracle.ainv(oracle.assemble(p), 0.1)
    off = M.nnz_offdiag
    assert bench.flop_model(p, "ainv", off, 2) == 2 * (2 * nnzA + 4 * (n + off) + n + 10 * n)
    assert bench.flop_model(p, "ainv", off, 1) - bench.flop_model(p, "jacobi", 0, 1) == 4 * (n + off)
