"""S = 3 / L = 2 block topology, batched on the GPU.

Reference: build_precoder / rzf_block / assemble_precoder (precoder.py:109-146),
assemble_blocks (channel.py:111-126), coupling_matrix and sinr_eq9
(metrics.py:35-58).  Per realization three independent RZF blocks -- side
subarray 1 for group 1 (M1 x K1), the central subarray for all users
(Mc x K), side subarray 2 for group 2 (M2 x K2) -- each with its own power
scaling beta (SPEC: per-block beta), stacked with exact zero blocks.

Batching: realizations with the same block shapes form one batch (the
reference's default topology always has K1 = K2 = K/2; ``group_by_shape``
buckets ragged draws).  Every block of a batch is one ``precode_batched``
call; the block coupling H^H G of the stacked matrices equals
H1^H G1 (+) Hc^H Gc (+) H2^H G2 exactly (the zero blocks add exact zeros,
test_metrics.py:39-44), so the SINR/SE runs through the same device kernel
as the single-block path.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import batched as BT
from .errors import ConfigurationError


def precode_batched(H: torch.Tensor, xi, power: float, method: str = "jacpcg", T: int = 5,
                    omega: float = 1.0, variant: str = "textbook", want_F: bool = False,
                    stream=None) -> BT.PrecoderBatch:
    """One RZF block per realization for any reference method (rzf_block,
    precoder.py:109-115): jacpcg / cg / direct through ``rzf_batched`` (fused
    when the shape allows), jor / gs through Gram -> stationary solve -> F = H X."""
    if method in ("jacpcg", "cg", "direct"):
        return BT.rzf_batched(H, xi, power, method=method, T=T, variant=variant, want_gamma=False,
                              want_F=want_F, check=True, stream=stream)
    if method not in ("jor", "gs"):
        raise ConfigurationError(f"unknown solver {method!r}")
    A = BT.gram_batched(H, xi, stream=stream)
    X = BT.solve_batched(A, method, T=T, omega=omega, check=True, stream=stream).X
    return BT.apply_precoder_batched(H, X, power, want_F=want_F, check=True, stream=stream)


@dataclass
class BlockPrecoderBatch:
    """Batched mirror of BlockPrecoder (precoder.py:28-50)."""
    G1: torch.Tensor      # [B, M1, K1]
    Gc: torch.Tensor      # [B, Mc, K]
    G2: torch.Tensor      # [B, M2, K2]
    beta_1: torch.Tensor  # [B]
    beta_c: torch.Tensor
    beta_2: torch.Tensor
    G: torch.Tensor       # [B, M, K] stacked with exact zero blocks

    @property
    def K1(self) -> int:
        return self.G1.shape[2]


def _check_blocks(H1, Hc, H2):
    for t, n in ((H1, "H1"), (Hc, "Hc"), (H2, "H2")):
        if not isinstance(t, torch.Tensor) or t.dim() != 3:
            raise ConfigurationError(f"{n} must be a [B, rows, users] tensor")
    B, M1, K1 = H1.shape
    Bc, Mc, K = Hc.shape
    B2, M2, K2 = H2.shape
    if not (B == Bc == B2):
        raise ConfigurationError("block batches differ in size")
    if K != K1 + K2:  # AssemblyError in the reference (channel.py:117-119)
        raise ConfigurationError(f"central block has {K} columns, expected K1+K2 = {K1 + K2}")
    return B, M1, Mc, M2, K1, K2, K


def assemble_blocks_batched(B1: torch.Tensor, Bc: torch.Tensor, B2: torch.Tensor) -> torch.Tensor:
    """Stack blocks into [B, M1+Mc+M2, K] with exact zero blocks (channel.py:111-126,
    precoder.py:118-133)."""
    B, M1, Mc, M2, K1, K2, K = _check_blocks(B1, Bc, B2)
    out = torch.zeros(B, M1 + Mc + M2, K, dtype=Bc.dtype, device=Bc.device)
    out[:, :M1, :K1] = B1
    out[:, M1:M1 + Mc, :] = Bc
    out[:, M1 + Mc:, K1:] = B2
    return out


def build_precoder_batched(H1: torch.Tensor, Hc: torch.Tensor, H2: torch.Tensor, xi, power: float,
                           method: str = "jacpcg", T: int = 5, omega: float = 1.0,
                           variant: str = "textbook", stream=None) -> BlockPrecoderBatch:
    """All three blocks of B realizations (build_precoder, precoder.py:136-146)."""
    _check_blocks(H1, Hc, H2)
    outs = [precode_batched(Hb, xi, power, method, T=T, omega=omega, variant=variant, stream=stream)
            for Hb in (H1, Hc, H2)]
    G1, Gc, G2 = (o.W for o in outs)
    return BlockPrecoderBatch(G1=G1, Gc=Gc, G2=G2, beta_1=outs[0].beta, beta_c=outs[1].beta,
                              beta_2=outs[2].beta, G=assemble_blocks_batched(G1, Gc, G2))


def block_sinr_batched(H1: torch.Tensor, Hc: torch.Tensor, H2: torch.Tensor,
                       pre: BlockPrecoderBatch, sigma2: float, stream=None) -> BT.SinrBatch:
    """sinr_eq9 on the block coupling (metrics.py:35-58) for B realizations."""
    H = assemble_blocks_batched(H1, Hc, H2)
    return BT.sinr_batched(H, pre.G.to(H.dtype), sigma2, stream=stream)


def group_by_shape(realizations) -> dict:
    """Bucket realizations (objects with H1 / Hc / H2) by block shapes:
    {(M1, Mc, M2, K1, K2): [indices]} -- each bucket is one batched call."""
    groups: dict = {}
    for i, r in enumerate(realizations):
        key = (*tuple(r.H1.shape), *tuple(r.Hc.shape[:1]), *tuple(r.H2.shape))
        groups.setdefault((key[0], key[2], key[3], key[1], key[4]), []).append(i)
    return groups
