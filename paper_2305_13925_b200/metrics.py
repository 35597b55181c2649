"""Reference-compatible link metrics (metrics.py:18-68), on the GPU.

``coupling_matrix`` / ``sinr_eq9`` accept the reference's realization and
precoder objects (anything with ``.H`` / ``.G``; the stacked block matrices
give exactly the block coupling, test_metrics.py:39-44) or plain (M, K)
arrays for one full-array block.  The arithmetic runs in xl_sinr.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import batched as BT
from .errors import ConfigurationError


@dataclass(frozen=True)
class LinkReport:
    gamma: np.ndarray        # (K,) per-user SINR
    se_per_user: np.ndarray  # (K,) log2(1 + gamma)
    sum_se: float
    noise_power: float


def _mat(x, attr):
    x = getattr(x, attr, x)
    if isinstance(x, torch.Tensor):
        return x
    return np.asarray(x)


def _pair(realization, precoder):
    H, G = _mat(realization, "H"), _mat(precoder, "G")
    to_np = not isinstance(H, torch.Tensor)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cuda"

    def dev_t(a):
        if isinstance(a, torch.Tensor):
            return a.to(dev).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex128))).to(dev)
    Hd, Gd = dev_t(H), dev_t(G)
    dt = torch.promote_types(Hd.dtype, Gd.dtype)
    if not dt.is_complex:
        dt = torch.complex128
    return Hd.to(dt)[None], Gd.to(dt)[None], to_np


def coupling_matrix(realization, precoder):
    """K x K effective gain matrix B = H^H G (metrics.py:35-44)."""
    Hd, Gd, to_np = _pair(realization, precoder)
    res = BT.sinr_batched(Hd, Gd, 1.0)
    B = res.coupling[0]
    return B.cpu().numpy() if to_np else B


def sinr_eq9(realization, precoder, sigma2: float) -> LinkReport:
    """Per-user SINR and SE (metrics.py:47-58)."""
    if sigma2 <= 0:
        raise ConfigurationError(f"noise power must be positive, got {sigma2}")
    Hd, Gd, _ = _pair(realization, precoder)
    res = BT.sinr_batched(Hd, Gd, sigma2)
    gamma = res.gamma[0].cpu().numpy()
    se = res.se[0].cpu().numpy()
    return LinkReport(gamma=gamma, se_per_user=se, sum_se=float(res.sum_se[0].item()),
                      noise_power=sigma2)


def sum_se(per_trial_sums) -> tuple[float, float]:
    """Monte-Carlo mean of per-trial sum SE and its standard error
    (metrics.py:61-68).  Device tensors reduce on the device in fixed chunk
    order; host sequences are tiny and reduce in numpy as in the reference."""
    if isinstance(per_trial_sums, torch.Tensor) and per_trial_sums.is_cuda:
        x = per_trial_sums.to(torch.float64).contiguous().reshape(-1)
        if x.numel() < 1:
            raise ConfigurationError("sum_se needs at least one trial")
        parts = BT.se_partials(x, 4096).cpu().numpy()
        return BT.combine_se_partials(parts)
    arr = np.asarray(per_trial_sums, dtype=float)
    if arr.size < 1:
        raise ConfigurationError("sum_se needs at least one trial")
    mean = float(arr.mean())
    sem = float(arr.std(ddof=1) / np.sqrt(arr.size)) if arr.size > 1 else 0.0
    return mean, sem
