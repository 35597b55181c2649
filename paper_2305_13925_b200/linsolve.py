"""Reference-compatible solver entry points (linsolve.py), run on the GPU.

Same names, arguments, return types and exceptions as
/root/reference/pkg/src/xlmimo/linsolve.py; the arithmetic runs in the
batched sm_100a solver (csrc/simt_solve.cu) with B = 1.  Numpy inputs are
promoted to complex128 exactly like the reference (linsolve.py:74, 222, 262);
a complex64 torch tensor keeps the fp32 path.

gs_solve / jor_solve run the stationary-splitting
kernel of the same file (xl_solve_stationary).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import batched as BT
from .errors import ConfigurationError, NotHpdError, SplittingError

HERMITIAN_RTOL = 1e-12


@dataclass(frozen=True)
class HpdSystem:
    """A Hermitian positive-definite matrix with right-hand side(s)
    (linsolve.py:21-43, same validation)."""

    P: np.ndarray
    rhs: np.ndarray
    xi: float | None = None

    def __post_init__(self):
        P = np.asarray(self.P)
        if P.ndim != 2 or P.shape[0] != P.shape[1]:
            raise NotHpdError(f"P must be square, got shape {P.shape}")
        rhs = np.asarray(self.rhs)
        if rhs.shape[0] != P.shape[0] or rhs.ndim not in (1, 2):
            raise NotHpdError(f"rhs shape {rhs.shape} incompatible with n={P.shape[0]}")
        scale = max(1.0, float(np.abs(P).max()))
        if not np.allclose(P, P.conj().T, atol=HERMITIAN_RTOL * scale, rtol=0):
            raise NotHpdError("P is not Hermitian to machine precision")

    @property
    def n(self) -> int:
        return self.P.shape[0]


@dataclass
class SolverOutcome:
    """Solution, iteration count, residual telemetry, convergence flag
    (linsolve.py:60-68)."""

    w: np.ndarray
    iterations: int
    residual_trace: np.ndarray
    converged: bool
    iterates: list = field(default_factory=list)


def _device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None


def _to_dev(x, dt):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=dt))).to(_device())


def _run(sys: HpdSystem, method, T, eps=None, w0=None, precond=None, precond_identity=False,
         keep_iterates=False, variant="textbook", omega=0.5) -> SolverOutcome:
    s = np.asarray(sys.rhs, dtype=complex)
    was_1d = s.ndim == 1
    s2 = s[:, None] if was_1d else s
    if w0 is not None:
        w = np.asarray(w0, dtype=complex)
        w = w[:, None] if w.ndim == 1 else w
        if w.shape != s2.shape:
            raise ConfigurationError(f"w0 shape {w.shape} does not match rhs shape {s2.shape}")
        w0 = w
    dt = np.complex128
    A = _to_dev(sys.P, dt)[None]
    S = _to_dev(s2, dt)[None]
    W0 = _to_dev(w0, dt)[None] if w0 is not None else None
    C = torch.from_numpy(np.asarray(precond, dtype=np.float64))[None].to(A.device) if precond is not None else None
    res = BT.solve_batched(A, method, T=max(T, 1), variant=variant, S=S, w0=W0, precond=C,
                           precond_identity=precond_identity, eps=eps, trace=True,
                           iterates=keep_iterates, check=True, omega=omega)
    its = int(res.iterations[0].item())
    trace = res.trace[0].cpu().numpy()[: (its + 1) if method != "direct" else 1]
    X = res.X[0].cpu().numpy()
    iterates = []
    if keep_iterates and its:
        arr = res.iterates[0, :its].cpu().numpy()
        iterates = [a[:, 0] if was_1d else a for a in arr]
    if method == "direct":
        converged = True
    elif eps is not None:
        converged = bool(np.sqrt(trace[-1]) <= eps)       # linsolve.py:103-106
    else:
        converged = bool(trace[-1] <= trace[0])
    return SolverOutcome(w=X[:, 0] if was_1d else X, iterations=its,
                         residual_trace=trace, converged=converged, iterates=iterates)


def direct_solve(sys: HpdSystem) -> SolverOutcome:
    """Exact Cholesky solve (linsolve.py:109-119)."""
    return _run(sys, "direct", 1)


def cg_solve(sys: HpdSystem, T: int, eps: float | None = None, w0=None,
             keep_iterates: bool = False) -> SolverOutcome:
    """Classical CG (linsolve.py:183-187)."""
    if T < 1:
        raise ConfigurationError(f"iteration count T must be >= 1, got {T}")
    return _run(sys, "cg", T, eps, w0, keep_iterates=keep_iterates)


def jacpcg_solve(sys: HpdSystem, T: int, eps: float | None = None, w0=None,
                 precond_diag=None, keep_iterates: bool = False,
                 variant: str = "algorithm") -> SolverOutcome:
    """Jacobi-preconditioned CG, C = diag(P) by default (linsolve.py:190-214)."""
    P = np.asarray(sys.P)
    if precond_diag is None:
        c = np.diag(P).real.copy()
    else:
        c = np.asarray(precond_diag, dtype=float).copy()
    if np.any(c == 0):
        raise SplittingError(f"preconditioner has zero diagonal entry at index "
                             f"{int(np.argmin(np.abs(c)))}")
    if variant not in ("algorithm", "textbook"):
        raise ConfigurationError(f"unknown PCG variant {variant!r}")
    if T < 1:
        raise ConfigurationError(f"iteration count T must be >= 1, got {T}")
    return _run(sys, "jacpcg", T, eps, w0, precond=c, keep_iterates=keep_iterates,
                variant=variant)


def _check_diag(P) -> None:
    """Zero diagonal entry -> SplittingError (linsolve.py:120-125)."""
    d = np.diag(np.asarray(P))
    if np.any(d == 0):
        raise SplittingError(f"zero diagonal entry at index {int(np.argmin(np.abs(d)))}")


def gs_solve(sys: HpdSystem, T: int, w0=None, eps: float | None = None,
             keep_iterates: bool = False) -> SolverOutcome:
    """Gauss-Seidel sweeps (D + Lo) w' = s - Up w (linsolve.py:128-151)."""
    if T < 1:
        raise ConfigurationError(f"iteration count T must be >= 1, got {T}")
    _check_diag(sys.P)
    return _run(sys, "gs", T, eps, w0, keep_iterates=keep_iterates)


def jor_solve(sys: HpdSystem, T: int, omega: float = 0.5, w0=None,
              eps: float | None = None, keep_iterates: bool = False) -> SolverOutcome:
    """Jacobi over-relaxation w <- w + omega D^-1 (s - P w) (linsolve.py:154-176)."""
    if T < 1:
        raise ConfigurationError(f"iteration count T must be >= 1, got {T}")
    if omega <= 0:
        raise ConfigurationError(f"relaxation omega must be positive, got {omega}")
    _check_diag(sys.P)
    return _run(sys, "jor", T, eps, w0, keep_iterates=keep_iterates, omega=omega)


ITERATIVE_SOLVERS = {  # linsolve.py:310-315
    "gs": gs_solve,
    "jor": jor_solve,
    "cg": cg_solve,
    "jacpcg": jacpcg_solve,
}
