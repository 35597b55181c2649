"""Multi-process (gloo, world_size 2, CPU) tests of the realization sharding
and the ergodic-SE reduction (distributed.py; reference sum_se,
metrics.py:61-68).

The per-realization sum-SE values come from the CPU oracle here (the device
kernels need a GPU); the chunk partials follow the xl_se_partials contract
({sum x, sum x^2, n} per `chunk` consecutive realizations, index order).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import xlmimo_oracle as O
from paper_2305_13925_b200 import distributed as D

TOTAL, CHUNK = 13, 4           # ragged: uneven shards and a partial last chunk
S, K, P, R = 1, 4, 0.7, 0.5    # tiny channels (M = 64) so the oracle is instant


def _sum_se_oracle(first, count):
    if count == 0:
        return np.zeros(0)
    H = O.generate_channels(0, first, count, S, K, P, R)
    return np.array([O.precoder_and_se(h, K / 10.0, 10.0, 1.0, "jacpcg", 4, "textbook")[3] for h in H])


def _partials(x, chunk):
    out = []
    for c0 in range(0, len(x), chunk):
        v = x[c0:c0 + chunk]
        out.append([v.sum(), (v * v).sum(), float(len(v))])
    return torch.tensor(out, dtype=torch.float64).reshape(-1, 3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, count = D.shard_range(TOTAL, world, rank)
        x = _sum_se_oracle(first, count)
        # chunks are per rank (index order inside the shard), like the bench
        parts = _partials(x, CHUNK)
        allp = D.gather_partials(parts)
        mean, sem = D.combine_partials_device(allp)
        out[rank] = (first, count, float(mean), float(sem), allp.shape[0])
        # the public combine path on ragged shards (the shards
        # hold different chunk counts; gather_partials pads them)
        m2, s2 = D.ergodic_from_partials(parts)
        out[world + rank] = (float(m2), float(s2))
        # the public entry point with group=False never communicates
        m3, _ = D.ergodic_from_partials(parts, group=False)
        out[2 * world + rank] = float(m3)
        # bench timing helpers: barrier + timed region + max over ranks
        import time
        with D.DeviceTimer("cpu") as t:
            time.sleep(0.05 + 0.15 * rank)
        out[3 * world + rank] = (t.ms, D.max_over_ranks([rank + 1.0, 10.0 - rank]))
    finally:
        dist.destroy_process_group()


def test_shard_range_covers_exactly_once():
    for total in (0, 1, 7, 13, 32768):
        for world in (1, 2, 3, 8):
            got = [D.shard_range(total, world, r) for r in range(world)]
            assert sum(c for _, c in got) == total
            pos = 0
            for f, c in got:
                assert f == pos
                pos += c


def test_combine_partials_matches_sum_se():
    x = _sum_se_oracle(0, TOTAL)
    mean, sem = D.combine_partials_device(_partials(x, CHUNK))
    rm, rs = O.sum_se(x)
    assert abs(float(mean) - rm) <= 1e-12 * abs(rm)
    assert abs(float(sem) - rs) <= 1e-9 * rs
    one = D.combine_partials_device(_partials(x[:1], CHUNK))
    assert float(one[1]) == 0.0  # SEM of a single trial is 0 (metrics.py:66-67)


@pytest.mark.timeout(300)
def test_gloo_two_ranks_ergodic_se():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    x = _sum_se_oracle(0, TOTAL)
    rm, rs = O.sum_se(x)
    for r in range(world):
        first, count, mean, sem, nchunks = out[r]
        assert (first, count) == D.shard_range(TOTAL, world, r)
        # every rank holds the same global result, equal to the single-process one
        assert abs(mean - rm) <= 1e-12 * abs(rm), (mean, rm)
        assert abs(sem - rs) <= 1e-9 * rs, (sem, rs)
        assert nchunks == sum(-(-D.shard_range(TOTAL, world, q)[1] // CHUNK) for q in range(world))
    assert out[0][2:4] == out[1][2:4]  # bit-identical on both ranks
    for r in range(world):
        assert abs(out[world + r][0] - rm) <= 1e-12 * abs(rm)
        assert abs(out[world + r][1] - rs) <= 1e-9 * rs
        ms, mx = out[3 * world + r]
        assert ms >= 200.0 * 0.9, ms          # the slower rank's 0.2 s on every rank
        assert mx == [2.0, 10.0]
    # rank-local combine sees only its own shard
    m0 = O.sum_se(x[:D.shard_range(TOTAL, world, 0)[1]])[0]
    assert abs(out[2 * world] - m0) <= 1e-12 * abs(m0)


def test_rank_batch_weak_and_strong():
    assert [D.rank_batch("weak", 100, 4, r) for r in range(4)] == [(0, 100), (100, 100), (200, 100), (300, 100)]
    got = [D.rank_batch("strong", 32768, 8, r) for r in range(8)]
    assert got[0] == (0, 4096) and got[7] == (28672, 4096)
    assert sum(c for _, c in [D.rank_batch("strong", 4097, 2, r) for r in range(2)]) == 4097
    with pytest.raises(ValueError):
        D.rank_batch("other", 1, 1, 0)
