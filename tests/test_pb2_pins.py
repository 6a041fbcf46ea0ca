"""Pins for the oracle's P_B2 (NEXT-4): Bridson-style AINV with a predetermined number of
nonzeros per column (reading R26).  Checked against the
limits SPEC states (m >= n reproduces tau = 0, m = 1 is the diagonal factor), the second
(dense right-looking) formulation, the count bound, SPD-ness and monotonicity in m.
Runs without a GPU."""
import numpy as np
import pytest

import oracle
from paper_1210_1878_b200 import synth

INF = float("inf")


def same(M1, M2):
    return (np.array_equal(M1.colptr, M2.colptr) and np.array_equal(M1.row, M2.row)
            and np.array_equal(M1.zhat, M2.zhat) and np.array_equal(M1.pivots, M2.pivots))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_fill_n_is_tau0_and_fill1_is_diagonal(seed):
    """m >= n reproduces tau = 0; m = 1 -> diagonal factor (= tau = inf)."""
    A = oracle.assemble(synth.random_grid(9, 8, seed))
    assert same(oracle.ainv(A, 0.0, fill=A.n), oracle.ainv(A, 0.0))
    M1 = oracle.ainv(A, 0.0, fill=1)
    assert same(M1, oracle.ainv(A, INF))
    assert np.all(np.diff(M1.colptr) == 1)


@pytest.mark.parametrize("fill", [2, 3, 5, 8])
@pytest.mark.parametrize("shape", [(8, 7, 1), (9, 8, 2), (12, 6, 3)])
@pytest.mark.parametrize("tau", [0.0, 0.05 + 1e-9])
def test_sparse_equals_dense_bitwise(fill, shape, tau):
    """Left-looking sparse and right-looking dense A-orthogonalisation apply the same update
    sequence per column, so with the count rule after every update they agree bit for bit."""
    ni, nj, seed = shape
    A = oracle.assemble(synth.random_grid(ni, nj, seed))
    Ms = oracle.ainv(A, tau, fill=fill)
    Md = oracle.ainv(A, tau, method="dense", fill=fill)
    assert same(Ms, Md)
    assert np.all(np.diff(Ms.colptr) <= fill)


def test_cfg1_ties_sparse_equals_dense():
    """cfg1 (constant couplings) has exact magnitude ties: the deterministic tie rule (smaller
    row index) makes both formulations agree bitwise there too."""
    A = oracle.assemble(synth.config("cfg1"))
    for fill in (2, 3, 4):
        assert same(oracle.ainv(A, 0.0, fill=fill), oracle.ainv(A, 0.0, method="dense", fill=fill))


def test_spd_and_iterations_monotone_in_fill():
    """cfg2: P = Z D^-1 Z^T is symmetric positive; PCG converges for every m, and more fill
    never needs more iterations over m = 1, 2, 4, 8, 16 (Jacobi at m = 1)."""
    p = synth.config("cfg2")
    A = oracle.assemble(p)
    b = A.apply(A.from_grid(synth.xstar(p)))
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(A.n), rng.standard_normal(A.n)
    its = []
    for m in (1, 2, 4, 8, 16):
        M = oracle.ainv(A, 0.0, fill=m)
        px, py = M.apply(x), M.apply(y)
        assert abs(px @ y - x @ py) <= 1e-12 * abs(px @ y) and x @ px > 0
        r = oracle.pcg(A, b, "ainv", M, 1e-10, maxit=5000)
        assert r.converged
        its.append(r.iterations)
    jac = oracle.pcg(A, b, "jacobi", None, 1e-10, maxit=5000).iterations
    assert its[0] == jac
    assert all(its[i + 1] <= its[i] for i in range(len(its) - 1))
