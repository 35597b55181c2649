"""Convergence telemetry and the BER detection chain on the GPU
(reference metrics.py:93-185).

The reference's ``convergence_trace`` and ``ber_montecarlo`` wrap per-trial
loops around a configuration object, a scenario generator and numpy RNG
streams (its control plane, out of scope here).  What runs per trial is
batched here over many channel draws at once:

* ``convergence_traces_batched`` -- regularized Gram of each draw's channel,
  the named iterative solver on one right-hand side per draw with residual
  telemetry, each trace held at its final value after an early Krylov stop
  (metrics.py:172-184); ``median_trace`` is the reference's per-iteration
  ``np.median`` over trials.
* ``ber_errors_batched`` -- Y = Bc s + n, genie scaling by the diagonal gain,
  hard QPSK decisions and the bit-error count per draw (metrics.py:124-140),
  one CUDA kernel (csrc/link_ber.cu) behind ``xl_ber_errors``.
* ``ber_point_batched`` -- one SNR point for several methods on the same
  draws (paired, like metrics.py:126-139): precoder per method on the device,
  coupling B = H^H G, then the detection chain.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import batched as BT
from .errors import ConfigurationError


def qpsk_modulate(bits):
    """Bit pairs (..., 2) -> ((1-2b0) + j(1-2b1))/sqrt(2) (metrics.py:73-77)."""
    bits = np.asarray(bits)
    return ((1.0 - 2.0 * bits[..., 0]) + 1j * (1.0 - 2.0 * bits[..., 1])) / np.sqrt(2.0)


def qpsk_detect(y):
    """Hard decisions back to bit pairs (metrics.py:80-83)."""
    y = np.asarray(y)
    return np.stack([(y.real < 0).astype(np.int8), (y.imag < 0).astype(np.int8)], axis=-1)


def convergence_traces_batched(H: torch.Tensor, xi, S: torch.Tensor, methods, T_max: int,
                               omega: float = 1.0, variant: str = "textbook",
                               stream=None) -> dict:
    """Per-draw residual traces ||P w_t - s||^2 / ||s||^2, t = 0..T_max, of each
    method on P = H^H H + xi I (metrics.py:165-184).  H [B, M, K] (the central
    subarray channels), S [B, K] right-hand sides.  Returns {method: [B, T_max+1]}
    float64 device tensors, held at the final value after an early stop."""
    methods = [m for m in methods if m != "direct"]
    if not methods:
        raise ConfigurationError("convergence trace needs at least one iterative method")
    if T_max < 1:
        raise ConfigurationError(f"T_max must be >= 1, got {T_max}")
    B, M, K = H.shape
    if tuple(S.shape) != (B, K):
        raise ConfigurationError(f"S must be [B, K] = {(B, K)}, got {tuple(S.shape)}")
    A = BT.gram_batched(H, xi, stream=stream)
    Sd = S.to(device=H.device, dtype=H.dtype).reshape(B, K, 1).contiguous()
    t = torch.arange(T_max + 1, device=H.device)
    out = {}
    for m in methods:
        r = BT.solve_batched(A, m, T=T_max, variant=variant, S=Sd, trace=True, omega=omega,
                             check=True, stream=stream)
        its = r.iterations.to(torch.int64)
        last = r.trace.gather(1, its[:, None])
        out[m] = torch.where(t[None, :] <= its[:, None], r.trace, last)
    return out


def median_trace(traces: torch.Tensor) -> np.ndarray:
    """np.median over trials (axis 0), as metrics.py:185: the mean of the two
    middle values for an even count."""
    x = torch.sort(traces.to(torch.float64), dim=0).values
    n = x.shape[0]
    if n % 2:
        return x[n // 2].cpu().numpy()
    return ((x[n // 2 - 1] + x[n // 2]) / 2.0).cpu().numpy()


def ber_errors_batched(Bc: torch.Tensor, bits: torch.Tensor, noise: torch.Tensor,
                       stream=None) -> torch.Tensor:
    """Bit errors per draw of the genie-scaled QPSK chain (metrics.py:124-140).
    Bc [B, K, K] coupling, bits [B, K, nsym, 2] int8 in {0, 1}, noise [B, K, nsym]."""
    lib = L.lib()
    BT._check_tensor(Bc, "Bc", 3)
    B, K, K2 = Bc.shape
    if K != K2:
        raise ConfigurationError("coupling must be square")
    if bits.dtype != torch.int8 or bits.dim() != 4 or tuple(bits.shape[:2]) != (B, K) or bits.shape[3] != 2:
        raise ConfigurationError("bits must be int8 [B, K, nsym, 2]")
    nsym = bits.shape[2]
    if tuple(noise.shape) != (B, K, nsym) or noise.dtype != Bc.dtype:
        raise ConfigurationError("noise must be [B, K, nsym] of the coupling dtype")
    bits = bits.to(Bc.device).contiguous()
    noise = noise.to(Bc.device).contiguous()
    err = torch.empty(B, dtype=torch.int64, device=Bc.device)
    rc = lib.xl_ber_errors(BT.dtype_code(Bc.dtype), L.ptr(Bc.contiguous()), L.ptr(bits), L.ptr(noise),
                           B, K, nsym, L.ptr(err), L.stream_ptr(stream))
    L.check(rc, "xl_ber_errors")
    return err


def ber_point_batched(H: torch.Tensor, xi, power: float, methods, bits: torch.Tensor,
                      noise: torch.Tensor, T: int = 5, omega: float = 1.0,
                      variant: str = "textbook", stream=None) -> dict:
    """One SNR point on B paired draws (metrics.py:124-140) with single-block
    precoders: {method: errors [B]}.  Iterative methods use rzf_batched
    (jacpcg / cg / direct) or the stationary solvers (jor / gs)."""
    from .blocks import precode_batched
    out = {}
    for m in methods:
        G = precode_batched(H, xi, power, m, T=T, omega=omega, variant=variant, stream=stream).W
        Bc = BT.sinr_batched(H, G, 1.0, stream=stream).coupling
        out[m] = ber_errors_batched(Bc, bits, noise, stream=stream)
    return out
