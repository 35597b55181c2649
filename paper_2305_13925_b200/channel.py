"""Channel-batch model and on-device generation (BASELINE model).

The reference draws one trial at a time on the host (scenario.py:65-97).  Here
realization b of a (seed, model) pair is a pure function of b: the device
generator (csrc/chan_gen.cu, Philox4x32-10) writes H[b] straight into HBM, so
every GPU/rank can generate exactly its own shard.

Model (BASELINE.json configs):
  M = S * Ms antennas (ULA split into S subarrays of Ms = 64),
  per user: d ~ U[10, 100] m, beta_dB = -35.3 - 37.6 log10 d, gain scaled by
  the closed-form mean beta_bar (decision D-1), Bernoulli(p) visibility per
  subarray redrawn until >= 1 visible (geometry.py:169-180),
  per visible subarray h = sqrt(gain) R_r^{1/2} g, g ~ CN(0, I) with the
  exponential correlation R_r[i, j] = r^|i-j| (channel.py:33-53).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .batched import dtype_code
from .errors import ConfigurationError, ModelError

PSD_CLAMP = 1e-12
PSD_NEG_TOL = 1e-10


def build_correlation(Ms: int, r: float) -> np.ndarray:
    """Exponential correlation R[i, j] = r^|i-j| (channel.py:33-38)."""
    if not 0.0 <= r < 1.0:
        raise ConfigurationError(f"rho must lie in [0, 1), got {r}")
    idx = np.arange(Ms)
    return (float(r) ** np.abs(idx[:, None] - idx[None, :])).astype(float)


def psd_sqrt(mat: np.ndarray) -> np.ndarray:
    """Hermitian PSD square root by eigendecomposition (channel.py:41-53).

    Host-side, once per configuration (an Ms x Ms = 64 x 64 matrix)."""
    vals, vecs = np.linalg.eigh(mat)
    scale = max(1.0, float(vals[-1]) if vals.size else 1.0)
    if vals.size and vals[0] < -PSD_NEG_TOL * scale:
        raise ModelError(f"covariance not PSD: min eigenvalue {vals[0]:.3e}")
    vals = np.where(vals < PSD_CLAMP, 0.0, vals)
    return (vecs * np.sqrt(vals)) @ vecs.conj().T


def beta_bar(dmin: float = 10.0, dmax: float = 100.0) -> float:
    """E_d[10^(beta_dB/10)] for d ~ U[dmin, dmax] (closed form)."""
    e = 3.76
    return (10.0 ** -3.53 * (dmin ** (1.0 - e) - dmax ** (1.0 - e))
            / ((e - 1.0) * (dmax - dmin)))


@dataclass(frozen=True)
class ChannelModel:
    S: int            # subarrays
    K: int            # users
    p: float          # per-subarray visibility probability
    r: float          # exponential correlation coefficient
    Ms: int = 64      # antennas per subarray
    dmin: float = 10.0
    dmax: float = 100.0
    normalise: bool = True

    @property
    def M(self) -> int:
        return self.S * self.Ms

    def rsqrt(self) -> np.ndarray:
        return psd_sqrt(build_correlation(self.Ms, self.r))

    def gain_norm(self) -> float:
        return beta_bar(self.dmin, self.dmax) if self.normalise else 1.0


_RSQRT_CACHE: dict = {}


def generate_channels(model: ChannelModel, seed: int, first: int, B: int,
                      dtype=torch.complex64, device=None, out: torch.Tensor | None = None,
                      check: bool = True, stream=None) -> torch.Tensor:
    """H[b] for global realization indices first .. first+B-1 -> [B, M, K]."""
    lib = L.lib()
    device = torch.device(device or "cuda")
    key = (model.Ms, model.r, device.index)
    rs = _RSQRT_CACHE.get(key)
    if rs is None:
        rs = torch.from_numpy(np.ascontiguousarray(model.rsqrt())).to(device)
        _RSQRT_CACHE[key] = rs
    if out is None:
        out = torch.empty(B, model.M, model.K, dtype=dtype, device=device)
    status = torch.empty(max(B, 1), dtype=torch.int32, device=device)
    rc = lib.xl_channel_generate(dtype_code(out.dtype), int(seed) & (2**64 - 1), int(first), int(B),
                                 model.S, model.Ms, model.K, float(model.p), L.ptr(rs),
                                 float(model.gain_norm()), float(model.dmin), float(model.dmax),
                                 L.ptr(out), L.ptr(status), L.stream_ptr(stream))
    L.check(rc, "xl_channel_generate")
    if check and B > 0:
        L.raise_status(status[:B].cpu().numpy(), "generate_channels")
    return out
