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


# ---- independent derivation of P_B2's kept set (VERDICT r1 "What's weak" 1) ----------------
# A dense right-looking A-orthogonalisation written here in plain Python floats (separate
# multiply and subtract, ascending sums -- the arithmetic of SURVEY §8(c.2)), with its OWN keep
# rule: numpy lexsort on (-|z|, row) -- largest magnitude first, ties to the smaller row index
# (R26).  Nothing of the oracle's selection code (sort comparator or the dense scan) is
# shared, so a wrong ordering or tie rule in the oracle fails here.
import math


def _py_ainv_fill(A, tau, fill, rule="R26"):
    rp, col, val = A.csr()
    n = A.n
    diag = np.array([val[e] for p in range(n) for e in range(rp[p], rp[p + 1]) if col[e] == p])
    s = [1.0 / math.sqrt(float(dp)) for dp in diag]
    rows = [[(int(col[e]), float(val[e]) * (s[p] * s[int(col[e])])) for e in range(rp[p], rp[p + 1])]
            for p in range(n)]
    Z = [{j: 1.0} for j in range(n)]
    piv = [0.0] * n
    ties = 0
    for i in range(n):
        zi = Z[i]
        pv = 0.0
        for k, a in rows[i]:
            if k in zi:
                pv = pv + a * zi[k]
        piv[i] = pv
        for j in range(i + 1, n):
            zj = Z[j]
            pi = 0.0
            for k, a in rows[i]:
                if k in zj:
                    pi = pi + a * zj[k]
            if pi == 0.0:
                continue
            c = pi / pv
            touched = []
            for k in sorted(zi):
                zj[k] = zj.get(k, 0.0) - c * zi[k]
                touched.append(k)
            for k in touched:
                if k != j and abs(zj[k]) < tau:
                    del zj[k]
            off = np.array(sorted(k for k in zj if k != j), dtype=np.int64)
            if fill > 0 and len(off) > fill - 1:
                mag = np.array([abs(zj[int(k)]) for k in off])
                if rule == "R26":          # largest first, ties to the smaller row
                    order = np.lexsort((off, -mag))
                elif rule == "ties_large":  # largest first, ties to the larger row
                    order = np.lexsort((-off, -mag))
                else:                       # "smallest": the wrong magnitude order
                    order = np.lexsort((off, mag))
                cut_in, cut_out = order[fill - 2] if fill >= 2 else None, order[fill - 1]
                if cut_in is not None and mag[cut_in] == mag[cut_out]:
                    ties += 1
                for k in off[order[fill - 1:]]:
                    del zj[int(k)]
    return Z, piv, ties


def _same_as_py(M, Z, piv):
    if not np.array_equal(M.pivots, np.array(piv)):
        return False
    for j in range(M.n):
        rows_j = M.row[M.colptr[j]:M.colptr[j + 1]]
        vals_j = M.zhat[M.colptr[j]:M.colptr[j + 1]]
        ks = sorted(Z[j])
        if list(rows_j) != ks or not np.array_equal(vals_j, np.array([Z[j][k] for k in ks])):
            return False
    return True


def _chain(n):
    """1-D chain of n unknowns (one ocean row, non-periodic), random couplings."""
    rng = np.random.default_rng(7)
    ocean = np.zeros((3, n), dtype=np.uint8)
    ocean[1, :] = 1
    cE = rng.uniform(0.5, 2.0, size=(3, n))
    cN = rng.uniform(0.5, 2.0, size=(3, n))
    cN[2, :] = 0.0
    return synth.Problem(f"chain{n}", n, 3, cE, cN, ocean, False, None)


def _const_grid(ni, nj):
    """Constant couplings (c = 1 on every face), land rows 0 and nj-1, E-W periodic: exact
    magnitude ties between mirror-image entries (at fill 3 one sits at the cut)."""
    ocean = np.ones((nj, ni), dtype=np.uint8)
    ocean[0, :] = 0
    ocean[nj - 1, :] = 0
    cE = np.ones((nj, ni))
    cN = np.ones((nj, ni))
    cN[nj - 1, :] = 0.0
    return synth.Problem(f"const{ni}x{nj}", ni, nj, cE, cN, ocean, True, None)


@pytest.mark.parametrize("fill", [2, 3])
@pytest.mark.parametrize("tau", [0.0, 0.05 + 1e-9])
@pytest.mark.parametrize("prob", ["chain", "grid6x5", "const6x5"])
def test_pb2_kept_set_independent(prob, tau, fill):
    p = {"chain": lambda: _chain(10), "grid6x5": lambda: synth.random_grid(6, 7, 4, land_frac=0.1),
         "const6x5": lambda: _const_grid(6, 7)}[prob]()
    A = oracle.assemble(p)
    Z, piv, _ = _py_ainv_fill(A, tau, fill)
    assert _same_as_py(oracle.ainv(A, tau, fill=fill), Z, piv)
    assert _same_as_py(oracle.ainv(A, tau, method="dense", fill=fill), Z, piv)


def test_pb2_pin_is_sensitive_to_the_rule():
    """The independent derivation must be able to fail: on the constant grid exact ties sit at
    the cut, so ties-to-the-larger-row gives another factor; keeping the smallest magnitudes
    gives another one on every problem."""
    A = oracle.assemble(_const_grid(6, 7))
    Z, piv, ties = _py_ainv_fill(A, 0.0, 3)
    assert ties > 0
    M = oracle.ainv(A, 0.0, fill=3)
    assert _same_as_py(M, Z, piv)
    Zl, pl, _ = _py_ainv_fill(A, 0.0, 3, rule="ties_large")
    assert not _same_as_py(M, Zl, pl)
    for prob in (_chain(10), synth.random_grid(6, 7, 4, land_frac=0.1)):
        A = oracle.assemble(prob)
        Zs, ps, _ = _py_ainv_fill(A, 0.0, 2, rule="smallest")
        assert not _same_as_py(oracle.ainv(A, 0.0, fill=2), Zs, ps)
