"""CPU oracle for the Jac-PCG RZF precoding path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference simulator's hot path
(``/root/reference/pkg/src/xlmimo``).  It exists to *check* the CUDA product,
never to be the product: only ``tests/``, ``__graft_entry__.smoke()`` and the
CPU-baseline legs of ``bench.py`` may import it.  The product package
``paper_2305_13925_b200`` never imports anything under ``oracle/``.

Parity pin: every function below is validated against the reference package
itself by ``tests/golden/make_golden.py`` (which imports the live reference and
writes the committed fixtures ``tests/golden/*.npz``) and
``tests/test_oracle_golden.py`` (CPU).  All arithmetic is complex128 /
float64, exactly like the reference (``precoder.py:57``).

Citations are ``file:line`` relative to ``/root/reference/pkg/src/xlmimo``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg


class OracleError(Exception):
    """Raised where the reference raises an XlMimoError subclass.

    ``kind`` is the reference class name (``NotHpdError``, ``SplittingError``,
    ``DegenerateChannelError``, ``ConfigurationError``).
    """

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------------------
# linsolve.py restatement
# ---------------------------------------------------------------------------

@dataclass
class Outcome:
    """Mirror of ``SolverOutcome`` (linsolve.py:60-68)."""

    w: np.ndarray
    iterations: int
    residual_trace: np.ndarray
    converged: bool
    iterates: list = field(default_factory=list)


def _prepare(rhs, w0):
    """linsolve.py:71-86."""
    s = np.asarray(rhs, dtype=complex)
    was_1d = s.ndim == 1
    s2 = s[:, None] if was_1d else s
    if w0 is None:
        w = np.zeros_like(s2)
    else:
        w = np.asarray(w0, dtype=complex)
        w = w[:, None] if w.ndim == 1 else w
        if w.shape != s2.shape:
            raise OracleError("ConfigurationError", "w0 shape mismatch")
        w = w.copy()
    snorm2 = float(np.vdot(s2, s2).real)
    return s2, w, was_1d, (snorm2 if snorm2 > 0 else 1.0)


def _ls_error(P, w, s2, snorm2):
    """linsolve.py:89-91."""
    r = P @ w - s2
    return float(np.vdot(r, r).real / snorm2)


def _finish(w, was_1d, iterations, trace, converged, iterates):
    """linsolve.py:94-100."""
    w_out = w[:, 0] if was_1d else w
    if was_1d:
        iterates = [x[:, 0] for x in iterates]
    return Outcome(w_out, iterations, np.asarray(trace), converged, iterates)


def _converged_flag(trace, eps):
    """linsolve.py:103-106."""
    if eps is not None:
        return bool(np.sqrt(trace[-1]) <= eps)
    return bool(trace[-1] <= trace[0])


def _col_dot(a, b):
    """linsolve.py:179-180."""
    return np.einsum("ij,ij->j", a.conj(), b).real


def direct_solve(P, rhs):
    """linsolve.py:109-119 (Cholesky + cho_solve)."""
    s2, _, was_1d, snorm2 = _prepare(rhs, None)
    try:
        factor = scipy.linalg.cho_factor(np.asarray(P, dtype=complex), lower=True)
    except (np.linalg.LinAlgError, scipy.linalg.LinAlgError) as exc:
        raise OracleError("NotHpdError", f"Cholesky breakdown: {exc}") from exc
    w = scipy.linalg.cho_solve(factor, s2)
    trace = [_ls_error(P, w, s2, snorm2)]
    return _finish(w, was_1d, 0, trace, True, [])


def pcg_core(P, rhs, T, eps=None, w0=None, precond_diag=None,
             keep_iterates=False, variant="cg"):
    """linsolve.py:217-256: CG (variant='cg') and the paper's Algorithm 1
    (variant='pcg', recurrences on the preconditioned residual)."""
    if T < 1:
        raise OracleError("ConfigurationError", f"T must be >= 1, got {T}")
    P = np.asarray(P, dtype=complex)
    s2, w, was_1d, snorm2 = _prepare(rhs, w0)
    if variant == "pcg":
        c_col = precond_diag[:, None]
        r = (s2 - P @ w) / c_col
    else:
        r = s2 - P @ w
    m = r.copy()
    rr = _col_dot(r, r)
    trace = [_ls_error(P, w, s2, snorm2)]
    iterates = []
    it = 0
    for t in range(1, T + 1):
        if not np.any(rr > 0):
            break
        Pm = P @ m
        z = (Pm / c_col) if variant == "pcg" else Pm
        curv = _col_dot(m, z)
        if np.any((curv <= 0) & (rr > 0)):
            raise OracleError("NotHpdError", "nonpositive curvature")
        alpha = np.where(rr > 0, rr / np.where(curv > 0, curv, 1.0), 0.0)
        w = w + alpha * m
        r = r - alpha * z
        rr_new = _col_dot(r, r)
        beta = np.where(rr > 0, rr_new / np.where(rr > 0, rr, 1.0), 0.0)
        m = r + beta * m
        rr = rr_new
        it = t
        trace.append(_ls_error(P, w, s2, snorm2))
        if keep_iterates:
            iterates.append(w.copy())
        if eps is not None and np.sqrt(trace[-1]) <= eps:
            break
    return _finish(w, was_1d, it, trace, _converged_flag(trace, eps), iterates)


def pcg_textbook(P, rhs, T, c, eps=None, w0=None, keep_iterates=False):
    """linsolve.py:259-294: standard PCG with r^H z inner products."""
    if T < 1:
        raise OracleError("ConfigurationError", f"T must be >= 1, got {T}")
    P = np.asarray(P, dtype=complex)
    s2, w, was_1d, snorm2 = _prepare(rhs, w0)
    c_col = c[:, None]
    r = s2 - P @ w
    z = r / c_col
    m = z.copy()
    rz = np.einsum("ij,ij->j", r.conj(), z).real
    trace = [_ls_error(P, w, s2, snorm2)]
    iterates = []
    it = 0
    for t in range(1, T + 1):
        if not np.any(rz > 0):
            break
        Pm = P @ m
        curv = _col_dot(m, Pm)
        if np.any((curv <= 0) & (rz > 0)):
            raise OracleError("NotHpdError", "nonpositive curvature")
        alpha = np.where(rz > 0, rz / np.where(curv > 0, curv, 1.0), 0.0)
        w = w + alpha * m
        r = r - alpha * Pm
        z = r / c_col
        rz_new = np.einsum("ij,ij->j", r.conj(), z).real
        beta = np.where(rz > 0, rz_new / np.where(rz > 0, rz, 1.0), 0.0)
        m = z + beta * m
        rz = rz_new
        it = t
        trace.append(_ls_error(P, w, s2, snorm2))
        if keep_iterates:
            iterates.append(w.copy())
        if eps is not None and np.sqrt(trace[-1]) <= eps:
            break
    return _finish(w, was_1d, it, trace, _converged_flag(trace, eps), iterates)


def cg_solve(P, rhs, T, eps=None, w0=None, keep_iterates=False):
    """linsolve.py:183-187."""
    return pcg_core(P, rhs, T, eps, w0, None, keep_iterates, "cg")


def jacpcg_solve(P, rhs, T, eps=None, w0=None, precond_diag=None,
                 keep_iterates=False, variant="algorithm"):
    """linsolve.py:190-214."""
    P = np.asarray(P)
    if precond_diag is None:
        c = np.diag(P).real.copy()
    else:
        c = np.asarray(precond_diag, dtype=float).copy()
    if np.any(c == 0):
        raise OracleError("SplittingError", "zero preconditioner diagonal")
    if variant not in ("algorithm", "textbook"):
        raise OracleError("ConfigurationError", f"unknown variant {variant!r}")
    if variant == "textbook":
        return pcg_textbook(P, rhs, T, c, eps, w0, keep_iterates)
    return pcg_core(P, rhs, T, eps, w0, c, keep_iterates, "pcg")


# ---------------------------------------------------------------------------
# precoder.py / metrics.py restatement
# ---------------------------------------------------------------------------

def _check_diag(P):
    """linsolve.py:120-125: exact zero on the (complex) diagonal."""
    d = np.diag(P)
    if np.any(d == 0):
        raise OracleError("SplittingError", f"zero diagonal entry at index {int(np.argmin(np.abs(d)))}")
    return d


def gs_solve(P, rhs, T, w0=None, eps=None, keep_iterates=False):
    """linsolve.py:128-151: Gauss-Seidel, w' = (D + Lo)^{-1} (s - Up w).

    The reference calls scipy's solve_triangular; this restatement does the
    forward substitution explicitly (row i: w_i = (r_i - sum_{l<i} P_il w_l) / P_ii).
    """
    if T < 1:
        raise OracleError("ConfigurationError", f"iteration count T must be >= 1, got {T}")
    P = np.asarray(P, dtype=complex)
    _check_diag(P)
    s2, w, was_1d, snorm2 = _prepare(rhs, w0)
    n = P.shape[0]
    Up = np.triu(P, 1)
    trace = [_ls_error(P, w, s2, snorm2)]
    iterates, it = [], 0
    for t in range(1, T + 1):
        r = s2 - Up @ w
        wn = np.empty_like(r)
        for i in range(n):
            wn[i] = (r[i] - P[i, :i] @ wn[:i]) / P[i, i]
        w = wn
        it = t
        trace.append(_ls_error(P, w, s2, snorm2))
        if keep_iterates:
            iterates.append(w.copy())
        if eps is not None and np.sqrt(trace[-1]) <= eps:
            break
    return _finish(w, was_1d, it, trace, _converged_flag(trace, eps), iterates)


def jor_solve(P, rhs, T, omega=0.5, w0=None, eps=None, keep_iterates=False):
    """linsolve.py:154-176: Jacobi over-relaxation w <- w + omega (s - P w) / d."""
    if T < 1:
        raise OracleError("ConfigurationError", f"iteration count T must be >= 1, got {T}")
    if omega <= 0:
        raise OracleError("ConfigurationError", f"relaxation omega must be positive, got {omega}")
    P = np.asarray(P, dtype=complex)
    d = _check_diag(P)[:, None]
    s2, w, was_1d, snorm2 = _prepare(rhs, w0)
    trace = [_ls_error(P, w, s2, snorm2)]
    iterates, it = [], 0
    for t in range(1, T + 1):
        w = w + omega * ((s2 - P @ w) / d)
        it = t
        trace.append(_ls_error(P, w, s2, snorm2))
        if keep_iterates:
            iterates.append(w.copy())
        if eps is not None and np.sqrt(trace[-1]) <= eps:
            break
    return _finish(w, was_1d, it, trace, _converged_flag(trace, eps), iterates)


def gram_regularized(H, xi):
    """precoder.py:53-61: P = H^H H + xi I, symmetrised; rhs = I."""
    if xi <= 0:
        raise OracleError("ConfigurationError", "xi must be positive")
    H = np.asarray(H, dtype=complex)
    n = H.shape[1]
    P = H.conj().T @ H + xi * np.eye(n)
    P = (P + P.conj().T) / 2.0
    return P


def power_scale(F, power):
    """precoder.py:64-70: beta = sqrt(power / ||F||_F^2), G = beta F."""
    tr = float(np.vdot(F, F).real)
    if tr <= 0:
        raise OracleError("DegenerateChannelError", "tr(F^H F) = 0")
    beta = float(np.sqrt(power / tr))
    return beta * F, F, beta


def rzf_direct(H, xi, power):
    """precoder.py:73-78."""
    P = gram_regularized(H, xi)
    Pinv = direct_solve(P, np.eye(P.shape[0], dtype=complex)).w
    F = np.asarray(H, dtype=complex) @ Pinv
    return power_scale(F, power)


def rzf_iterative(H, xi, power, solver="jacpcg", T=5, eps=None,
                  pcg_variant="algorithm"):
    """precoder.py:81-91 (+ solve_iterative 94-106 for cg/jacpcg)."""
    if T < 1:
        raise OracleError("ConfigurationError", "T must be >= 1")
    P = gram_regularized(H, xi)
    I = np.eye(P.shape[0], dtype=complex)
    if solver == "jacpcg":
        out = jacpcg_solve(P, I, T, eps=eps, variant=pcg_variant)
    elif solver == "cg":
        out = cg_solve(P, I, T, eps=eps)
    else:
        raise OracleError("ConfigurationError", f"unknown solver {solver!r}")
    F = np.asarray(H, dtype=complex) @ out.w
    return power_scale(F, power)


def sinr_single_block(H, G, sigma2):
    """metrics.py:47-58 on one full-array block.

    The reference's ``coupling_matrix`` (metrics.py:35-44) with empty side
    blocks reduces to B = H^H G (pinned at test_metrics.py:39-44).
    Returns (gamma, se_per_user, sum_se).
    """
    if sigma2 <= 0:
        raise OracleError("ConfigurationError", "sigma2 must be positive")
    B = np.asarray(H, dtype=complex).conj().T @ np.asarray(G, dtype=complex)
    diag = np.diag(B)
    signal = np.abs(diag) ** 2
    interference = np.sum(np.abs(B) ** 2, axis=1) - signal
    gamma = signal / (interference + sigma2)
    se = np.log2(1.0 + gamma)
    return gamma, se, float(se.sum())


def sum_se(per_trial_sums):
    """metrics.py:61-68: Monte-Carlo mean and SEM (ddof=1)."""
    arr = np.asarray(per_trial_sums, dtype=float)
    if arr.size < 1:
        raise OracleError("ConfigurationError", "need at least one trial")
    mean = float(arr.mean())
    sem = float(arr.std(ddof=1) / np.sqrt(arr.size)) if arr.size > 1 else 0.0
    return mean, sem


def precoder_and_se(H, alpha, power, sigma2, method="jacpcg", T=4,
                    variant="textbook"):
    """One realization of the hot path: (W, beta, gamma, sum_se).

    method: 'jacpcg' | 'cg' | 'direct'  (rzf_block, precoder.py:109-115).
    """
    if method == "direct":
        G, _, beta = rzf_direct(H, alpha, power)
    else:
        G, _, beta = rzf_iterative(H, alpha, power, method, T,
                                   pcg_variant=variant)
    gamma, _, s = sinr_single_block(H, G, sigma2)
    return G, beta, gamma, s


# ---------------------------------------------------------------------------
# flops.py restatement (integer closed forms, flops.py:35-69)
# ---------------------------------------------------------------------------

def flops_direct(K):
    return 4 * K ** 3 + K - 1


def flops_cg(K, T):
    return T * (8 * K ** 2 + 46 * K - 6)


def flops_jacpcg(K, T):
    return flops_cg(K, T) + (4 * K ** 2 + 2 * K)


# ---------------------------------------------------------------------------
# Channel-batch generator restatement (BASELINE model).
# Recipe follows scenario.py:85-88 (z ~ CN(0,1), R^{1/2} z, mask, scale),
# channel.py:33-53 (exponential correlation, PSD square root) and
# geometry.py:169-180 (resample until visible).  The random stream is
# Philox4x32-10 keyed by the master seed with counter (j, k|purpose<<24,
# b_lo, b_hi); the CUDA generator implements the same counter map.
# ---------------------------------------------------------------------------

_PH_M0 = np.uint64(0xD2511F53)
_PH_M1 = np.uint64(0xCD9E8D57)
_PH_W0 = np.uint32(0x9E3779B9)
_PH_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)

PURPOSE_DIST = 0
PURPOSE_VIS = 1
PURPOSE_FADE = 2
MAX_VIS_ATTEMPTS = 4096


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 (Salmon et al., SC'11) on broadcastable uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = _PH_M0 * c0.astype(np.uint64)
            p1 = _PH_M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK32).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32(k0 + _PH_W0)
            k1 = np.uint32(k1 + _PH_W1)
    return c0, c1, c2, c3


def _u01(x):
    """uint32 -> double in (0, 1): (x + 0.5) * 2^-32 (exact in binary64)."""
    return (np.asarray(x, dtype=np.float64) + 0.5) * (1.0 / 4294967296.0)


def correlation_sqrt(Ms, r):
    """psd_sqrt(build_correlation(Ms, r)) -- channel.py:33-53."""
    R = scipy.linalg.toeplitz(r ** np.arange(Ms)).astype(float)
    vals, vecs = np.linalg.eigh(R)
    vals = np.where(vals < 1e-12, 0.0, vals)
    return (vecs * np.sqrt(vals)) @ vecs.conj().T


def beta_bar(dmin=10.0, dmax=100.0, a=-35.3, b=-37.6):
    """Closed-form E_d[10^(beta_dB/10)], d ~ U[dmin, dmax]."""
    e = -b / 10.0  # path-loss exponent 3.76
    return (10.0 ** (a / 10.0) * (dmin ** (1.0 - e) - dmax ** (1.0 - e))
            / ((e - 1.0) * (dmax - dmin)))


def generate_channels(seed, first, B, S, K, p, r, Ms=64, dmin=10.0,
                      dmax=100.0, normalise=True, return_parts=False):
    """Batch of H[b] (M = S*Ms, K), complex128, b = first .. first+B-1.

    With ``return_parts`` also returns (amp[B,K], vis[B,K,S]).
    """
    k0 = np.uint32(seed & 0xFFFFFFFF)
    k1 = np.uint32((seed >> 32) & 0xFFFFFFFF)
    bidx = np.arange(first, first + B, dtype=np.uint64)
    b_lo = (bidx & _MASK32).astype(np.uint32)[:, None]
    b_hi = (bidx >> np.uint64(32)).astype(np.uint32)[:, None]
    users = np.arange(K, dtype=np.uint32)[None, :]

    # distance + large-scale gain
    x = philox4x32_10(np.uint32(0), users | np.uint32(PURPOSE_DIST << 24),
                      b_lo, b_hi, k0, k1)
    d = dmin + (dmax - dmin) * _u01(x[0])
    beta_db = -35.3 - 37.6 * np.log10(d)
    gain = 10.0 ** (beta_db / 10.0)
    if normalise:
        gain = gain / beta_bar(dmin, dmax)
    amp = np.sqrt(gain)                                     # (B, K)

    # visibility: Bernoulli(p) per subarray, redraw until >= 1 visible
    nq = (S + 3) // 4
    vis = np.zeros((B, K, S), dtype=bool)
    todo = np.ones((B, K), dtype=bool)
    for att in range(MAX_VIS_ATTEMPTS):
        if not todo.any():
            break
        cand = np.zeros((B, K, S), dtype=bool)
        for q in range(nq):
            y = philox4x32_10(np.uint32(att * nq + q),
                              users | np.uint32(PURPOSE_VIS << 24),
                              b_lo, b_hi, k0, k1)
            for e in range(4):
                s = 4 * q + e
                if s < S:
                    cand[:, :, s] = _u01(y[e]) < p
        ok = cand.any(axis=2) & todo
        vis[ok] = cand[ok]
        todo &= ~ok
    if todo.any():
        raise OracleError("GeometryInfeasibleError", "no visible subarray")

    # small-scale fading g ~ CN(0, 1): g = sqrt(-ln u1) e^{i 2 pi u2}
    half = Ms // 2
    j = np.arange(S * half, dtype=np.uint32)[None, None, :]
    z = philox4x32_10(j, users[:, :, None] | np.uint32(PURPOSE_FADE << 24),
                      b_lo[:, :, None], b_hi[:, :, None], k0, k1)
    g = np.empty((B, K, S * Ms), dtype=complex)
    for e in range(2):
        rad = np.sqrt(-np.log(_u01(z[2 * e])))
        th = 2.0 * np.pi * _u01(z[2 * e + 1])
        g[:, :, e::2] = rad * (np.cos(th) + 1j * np.sin(th))
    g = g.reshape(B, K, S, Ms)
    Rs = correlation_sqrt(Ms, r)
    hbar = np.einsum("ij,bksj->bksi", Rs, g)                # (B, K, S, Ms)
    h = hbar * vis[..., None] * amp[:, :, None, None]
    H = np.ascontiguousarray(h.reshape(B, K, S * Ms).transpose(0, 2, 1))
    if return_parts:
        return H, amp, vis
    return H
