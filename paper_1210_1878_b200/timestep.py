"""Time-stepping driver: NEMO's calling pattern of the elliptic solver.

NEMO-OPA advances the sea surface by leap-frog (Eq. 1) and solves the elliptic
system of Eq. 2 / Eq. 10 for D^{n+1} once per time step, with the same operator A (fixed grid,
depth and time step) and a new right-hand side.  So the setup (assembly, AINV, packing) is paid
once and every step is one pcg_solve, started from NEMO's first guess x0 = 2 D^n - D^{n-1}
(Alg. 1 l.1, reading R27) formed on the device by pcg_extrapolate.

This module only sequences library calls (pcg_solve, pcg_extrapolate, pcg_apply_operator); every
arithmetic step runs in libpcg's kernels.
"""
from __future__ import annotations

WARM = ("extrapolate", "previous", "zero")


class Stepper:
    """Repeated solves A D^{n+1} = b^{n+1} on one Solver, warm-started.

    warm = "extrapolate": x0 = 2 D^n - D^{n-1} (NEMO; "previous" for the first step),
           "previous":    x0 = D^n,
           "zero":        x0 = 0 (a cold solve every step)."""

    def __init__(self, solver, warm: str = "extrapolate"):
        if warm not in WARM:
            raise ValueError(f"warm must be one of {WARM}")
        self.S = solver
        self.warm = warm
        self.d_cur = None           # D^n
        self.d_prev = None          # D^{n-1}
        self.steps = 0

    def first_guess(self):
        if self.warm == "zero" or self.d_cur is None:
            return None
        if self.warm == "previous" or self.d_prev is None:
            return self.d_cur
        return self.S.extrapolate(self.d_cur, self.d_prev)

    def step(self, b, tol: float = 1e-10, maxit: int | None = None):
        """One time step: solve for D^{n+1} with right-hand side b (torch CUDA float64 [rows][ni]).
        Returns (D^{n+1}, iterations, report)."""
        x0 = self.first_guess()
        x, k, hist, rep = self.S.solve(b, x0=x0, tol=tol, maxit=maxit)
        self.d_prev, self.d_cur = self.d_cur, x
        self.steps += 1
        return x, k, rep
