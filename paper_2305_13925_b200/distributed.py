"""Multi-GPU realization sharding, device timing over ranks and the ergodic-SE
reduction.

The reference parallelises only over trials in a host process pool
(experiments.py:63-67).  Here realizations are sharded over GPUs (one process
per GPU, torch.distributed): rank g owns a contiguous range of global indices
(weak scaling: B per rank, [g B, (g + 1) B); strong scaling: ``shard_range``
of a fixed total) and generates its own channels from (seed, index) on device,
so there is no data-path exchange.  The only collective is the ergodic SE of
sum_se (metrics.py:61-68): every rank reduces its per-realization sum-SE into
fixed-size chunk partials {sum, sum^2, n} (xl_se_partials), the partials are
all-gathered (NCCL over NVLink/NVSwitch; 3 doubles per chunk; shards may be
ragged) and combined in global chunk order on every rank, so the result does
not depend on the GPU count.

Timing (bench.py): ``DeviceTimer`` brackets the timed steps with a barrier and
a device synchronize on both sides, times them with CUDA events on the
launching stream and takes the maximum over ranks (``max_over_ranks``).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def _active(group=None) -> bool:
    return (group is not False and dist.is_available() and dist.is_initialized()
            and dist.get_world_size(group if group else None) > 1)


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[first, first + count) of `total` realizations owned by `rank`
    (contiguous blocks, the first `total % world` ranks get one extra)."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def rank_batch(scaling: str, per_rank_or_total: int, world: int, rank: int) -> tuple[int, int]:
    """(first global index, count) of this rank's realizations.

    weak:   every rank owns ``per_rank_or_total`` realizations;
    strong: ``per_rank_or_total`` realizations in all, split by shard_range."""
    if scaling == "weak":
        return rank * per_rank_or_total, per_rank_or_total
    if scaling == "strong":
        return shard_range(per_rank_or_total, world, rank)
    raise ValueError(f"scaling must be 'weak' or 'strong', got {scaling!r}")


def combine_partials_device(parts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(mean, sem) as 0-d tensors from ordered [n_chunks, 3] partials (on a GPU:
    one xl_se_combine launch)."""
    if parts.is_cuda:
        from . import _lib as L
        parts = parts.contiguous()
        out = torch.empty(2, dtype=torch.float64, device=parts.device)
        L.check(L.lib().xl_se_combine(L.ptr(parts), parts.shape[0], L.ptr(out), L.stream_ptr(None)),
                "xl_se_combine")
        return out[0], out[1]
    s, q, n = parts[:, 0].sum(), parts[:, 1].sum(), parts[:, 2].sum()
    mean = s / n
    var = torch.clamp(q - n * mean * mean, min=0.0) / torch.clamp(n - 1.0, min=1.0)
    sem = torch.where(n > 1, torch.sqrt(var / n), torch.zeros_like(n))
    return mean, sem


def gather_partials(parts: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's chunk partials in rank (= global chunk) order.

    Shards may hold different numbers of chunks: the counts are gathered
    first and every rank pads to the largest, so each all_gather moves equal
    sizes (required by NCCL)."""
    world = dist.get_world_size(group)
    n = torch.tensor([parts.shape[0]], device=parts.device, dtype=torch.int64)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    counts = [int(s) for s in sizes]
    mx = max(counts)
    pad = torch.zeros(mx, 3, dtype=parts.dtype, device=parts.device)
    pad[: parts.shape[0]] = parts
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[r][: counts[r]] for r in range(world)])


def ergodic_from_partials(parts: torch.Tensor, group=None):
    """Mean/SEM over all ranks from this rank's ordered chunk partials.

    group=False forces the single-process path (no collective)."""
    if _active(group):
        parts = gather_partials(parts, group if group else None)
    return combine_partials_device(parts)


def ergodic_se(sum_se: torch.Tensor, chunk: int = 2048, group=None):
    """Ergodic SE mean/SEM over all ranks' realizations (device tensors).

    The chunk partials come from the xl_se_partials kernel; ragged shards
    (different chunk counts per rank) are handled by ``gather_partials``."""
    from . import batched as BT
    return ergodic_from_partials(BT.se_partials(sum_se, chunk), group)


def max_over_ranks(values, device=None, group=None) -> list[float]:
    """Element-wise maximum of per-rank floats (device-timed numbers)."""
    vals = [float(v) for v in values]
    if not _active(group):
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group if group else None)
    return [float(v) for v in t.tolist()]


def barrier(device=None, group=None):
    """Barrier over ranks (if any) followed by a device synchronize."""
    if _active(group):
        dist.barrier(group=group if group else None)
    if device is not None and torch.device(device).type == "cuda":
        torch.cuda.synchronize(device)


class DeviceTimer:
    """Barrier + synchronize on both sides of a timed region, CUDA events on
    the current stream inside it, and the maximum over ranks:

        with DeviceTimer(dev) as t:
            for _ in range(K): step()
        ms = t.ms          # max over ranks of the event-timed duration
    """

    def __init__(self, device, group=None):
        self.device, self.group = torch.device(device), group
        self.ms = None

    def __enter__(self):
        barrier(self.device, self.group)
        if self.device.type == "cuda":
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        else:
            import time
            self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        if exc[0] is not None:
            return False
        if self.device.type == "cuda":
            self.e1.record()
            torch.cuda.synchronize(self.device)
            ms = self.e0.elapsed_time(self.e1)
        else:
            import time
            ms = 1e3 * (time.perf_counter() - self.t0)
        barrier(self.device, self.group)
        self.ms = max_over_ranks([ms], self.device if self.device.type == "cuda" else None, self.group)[0]
        return False
