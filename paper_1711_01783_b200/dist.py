"""Multi-GPU plumbing of the decoder.

Frames are independent codewords, so the path shards without any data-path exchange:
frame f is decoded by rank f mod G (weak scaling).  The only collective is the
all-reduce of the per-batch frame counters written by metldpc_batch_counters
(north_star: "NCCL over NVLink is used only to gather per-frame convergence and FER
counts").  torch.distributed is plumbing here: NCCL on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

COUNTER_FIELDS = ("frames", "converged", "iterations", "invalid")


def shard_frames(frame_ids, rank: int, world: int):
    """The global frame ids decoded by `rank`: f with f mod world == rank, in order."""
    return [f for f in frame_ids if f % world == rank]


def reduce_counters(counters, group=None):
    """Sums the int64[4] counter tensor over ranks in place (NCCL / gloo all-reduce)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def summarize(counters) -> dict:
    frames, conv, iters, bad = (int(x) for x in counters)
    return {"frames": frames, "converged": conv, "fer": 1.0 - conv / max(1, frames),
            "mean_iters": iters / max(1, frames - bad), "invalid": bad}
