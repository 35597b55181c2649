"""An independent complex64 execution of the reference recurrences (numpy):
the round-off floor any complex64 implementation inherits.  Unpreconditioned
CG and the paper's Algorithm 1 amplify it beyond 1e-4 on some channels; their
c64 parity bound is stated against this."""

import numpy as np

from oracle import xlmimo_oracle as O


def relf(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _fp32_run(Hb, alpha, power, method, T, variant, coupling="hg"):
    """The same recurrences (linsolve.py:217-294) executed in complex64.

    Unpreconditioned CG and the paper's Algorithm-1 variant (which diverges
    on realistic channels) amplify fp32 round-off in their
    recurrences beyond 1e-4; no input perturbation models that, so the bound
    for those methods is how far an independent fp32 execution lands from
    the complex128 oracle."""
    f32, c64 = np.float32, np.complex64
    H = Hb.astype(c64)
    K = H.shape[1]
    P = H.conj().T @ H + f32(alpha) * np.eye(K, dtype=c64)
    c = np.diag(P).real.astype(f32)[:, None]
    dot = lambda a, b: np.einsum("ij,ij->j", a.conj(), b).real.astype(f32)
    w = np.zeros((K, K), c64)
    r = np.eye(K, dtype=c64)
    if method == "cg":
        z, m = r, r.copy()
    elif variant == "textbook":
        z = r / c
        m = z.copy()
    else:
        r = r / c
        z, m = r, r.copy()
    rz = dot(r, z)
    for _ in range(T):
        Pm = P @ m
        zz = Pm / c if (method == "jacpcg" and variant == "algorithm") else Pm
        a = np.where(rz > 0, rz / np.where(dot(m, zz) > 0, dot(m, zz), f32(1)), f32(0))
        w = w + a * m
        r = r - a * zz
        z = r / c if (method == "jacpcg" and variant == "textbook") else r
        rn = dot(r, z)
        m = z + np.where(rz > 0, rn / np.where(rz > 0, rz, f32(1)), f32(0)) * m
        rz = rn
    F = H @ w
    beta = np.sqrt(power / np.vdot(F, F).real)
    G = (beta * F).astype(c64)
    if coupling == "gx":  # B = beta (A - xi I) X in complex64: the K x K form the kernels use
        Bc = (f32(beta) * ((P - f32(alpha) * np.eye(K, dtype=c64)) @ w)).astype(np.complex128)
    else:                 # B = H^H G (metrics.py:35-44)
        Bc = (H.conj().T @ G).astype(np.complex128)
    sig = np.abs(np.diag(Bc)) ** 2
    intf = (np.abs(Bc) ** 2).sum(1) - sig
    return G, float(np.log2(1 + sig / (intf + 1.0)).sum())


def _fp32_sensitivity(Hb, alpha, power, method, T, variant):
    """(W, SE) relative distance of complex64 executions from the oracle: the
    SE distance is the larger of the two coupling formulations (H^H G, and
    the K x K beta (A - xi I) X the kernels use, metrics.py:35-44)."""
    G0, _, _, s0 = O.precoder_and_se(Hb, alpha, power, 1.0, method, T, variant)
    G1, s1 = _fp32_run(Hb, alpha, power, method, T, variant)
    _, s2 = _fp32_run(Hb, alpha, power, method, T, variant, coupling="gx")
    return relf(G1, G0), max(abs(s1 - s0), abs(s2 - s0)) / abs(s0)
