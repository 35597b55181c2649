"""Multi-GPU realization sharding and the ergodic-SE reduction.

The reference parallelises only over trials in a host process pool
(experiments.py:63-67).  Here realizations are sharded over GPUs (one process
per GPU, torch.distributed): rank g owns global indices
[g * B_local, (g + 1) * B_local) and generates its own channels from
(seed, index) on device, so there is no data-path exchange.  The only
collective is the ergodic SE of sum_se (metrics.py:61-68): every rank reduces
its per-realization sum-SE into fixed-size chunk partials {sum, sum^2, n}
(xl_se_partials), the partials are all-gathered (NCCL over NVLink/NVSwitch;
3 doubles per chunk) and combined in global chunk order on every rank.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import batched as BT


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[first, first + count) of `total` realizations owned by `rank`
    (contiguous blocks, the first `total % world` ranks get one extra)."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def combine_partials_device(parts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(mean, sem) as 0-d device tensors from ordered [n_chunks, 3] partials."""
    s, q, n = parts[:, 0].sum(), parts[:, 1].sum(), parts[:, 2].sum()
    mean = s / n
    var = torch.clamp(q - n * mean * mean, min=0.0) / torch.clamp(n - 1.0, min=1.0)
    sem = torch.where(n > 1, torch.sqrt(var / n), torch.zeros_like(n))
    return mean, sem


def gather_partials(parts: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's chunk partials in rank (= global chunk) order."""
    world = dist.get_world_size(group)
    n = torch.tensor([parts.shape[0]], device=parts.device, dtype=torch.int64)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(s) for s in sizes))
    pad = torch.zeros(mx, 3, dtype=parts.dtype, device=parts.device)
    pad[: parts.shape[0]] = parts
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[r][: int(sizes[r])] for r in range(world)])


def ergodic_se(sum_se: torch.Tensor, chunk: int = 2048, group=None):
    """Ergodic SE mean/SEM over all ranks' realizations (device tensors).

    group=False forces the single-process path (no collective)."""
    parts = BT.se_partials(sum_se, chunk)
    if group is not False and dist.is_available() and dist.is_initialized() \
            and dist.get_world_size(group if group else None) > 1:
        parts = gather_partials_fixed(parts, group if group else None)
    return combine_partials_device(parts)


def gather_partials_fixed(parts: torch.Tensor, group=None) -> torch.Tensor:
    """Equal-size shards (the benchmark case): one all_gather_into_tensor."""
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(parts) for _ in range(world)]
    dist.all_gather(bufs, parts.contiguous(), group=group)
    return torch.cat(bufs)
