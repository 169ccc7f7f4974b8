"""Multi-process (gloo, world size 2) tests of the sharding and counter aggregation
that bench.py uses over NCCL on GPUs."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_01783_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = D.shard_frames(range(10), rank, world)
        # per-rank counters as the k_counters kernel would write them: frames, converged,
        # sum of iterations over valid frames, invalid frames
        conv = sum(1 for f in frames if f % 3 == 0)
        iters = sum(100 if f % 3 else 7 for f in frames)
        c = torch.tensor([len(frames), conv, iters, 0], dtype=torch.int64)
        D.reduce_counters(c)
        t = D.max_over_ranks(1.0 + rank)
        out[rank] = (frames, c.tolist(), t)
    finally:
        dist.destroy_process_group()


def test_shard_frames_partition():
    ids = list(range(37))
    parts = [D.shard_frames(ids, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == ids
    assert all(f % 4 == r for r, p in enumerate(parts) for f in p)


def test_gloo_world2_counters_and_timing():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    frames0, c0, t0 = res[0]
    frames1, c1, t1 = res[1]
    assert frames0 == [0, 2, 4, 6, 8] and frames1 == [1, 3, 5, 7, 9]
    # totals equal the single-process sums over all frames
    conv = sum(1 for f in range(10) if f % 3 == 0)
    iters = sum(100 if f % 3 else 7 for f in range(10))
    assert c0 == c1 == [10, conv, iters, 0]
    assert t0 == t1 == 2.0           # max over ranks
    s = D.summarize(c0)
    assert s["frames"] == 10 and abs(s["fer"] - (1 - conv / 10)) < 1e-12
