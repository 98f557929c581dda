"""Multi-GPU plumbing (one process per GPU, torch.distributed) for the OSCAR hot path.

The path shards without a data-path collective:
  * quantize_append / attend are independent per (KV head, sequence): a rank owns a
    contiguous KV-head range for all sequences (`kv_head_shard`) or a batch slice
    (`batch_shard`), with its own pool, rotations and outputs;
  * calibration shards tokens (`token_shard`); the per-(layer, KV head) d x d covariance
    partial sums are then SUM-all-reduced (`allreduce_covariances`) — NCCL over NVLink /
    NVSwitch on B200 boxes, gloo in the CPU tests — before the eigensolver.
"""
from __future__ import annotations


def token_shard(n_tokens: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range [lo, hi) of calibration rows owned by `rank`."""
    base, rem = divmod(n_tokens, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def kv_head_shard(num_kv_heads: int, num_q_heads: int, rank: int, world: int):
    """(kv_lo, kv_hi, q_lo, q_hi): the KV heads of `rank` and their GQA query heads."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} KV heads cannot be split over {world} ranks")
    g = num_q_heads // num_kv_heads
    per = num_kv_heads // world
    return rank * per, (rank + 1) * per, rank * per * g, (rank + 1) * per * g


def batch_shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    return token_shard(batch, rank, world)


def allreduce_covariances(acc, world: int):
    """SUM the unnormalized covariance accumulators of all ranks in place (§3 targets are
    sums over tokens, so shard partials add exactly up to fp64 rounding)."""
    import torch.distributed as dist
    if world <= 1 and not (dist.is_available() and dist.is_initialized()):
        return acc
    dist.all_reduce(acc, op=dist.ReduceOp.SUM)       # (a 1-rank group still runs the collective)
    return acc


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(value: float, world: int) -> float:
    """Max of a per-rank scalar (device timings are reported as the max over ranks)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
