"""Multi-GPU sharding of the instance range.

The path is embarrassingly parallel over instances and strictly serial over
clocks, so rank d of D owns a contiguous block of whole 32-instance groups
and there is NO collective on the data path.  The only exchange is the
optional 8-byte end-of-run checksum: an all-reduce SUM of uint64 values (mod
2^64; NCCL has no XOR) carried as int64 through torch.distributed (NCCL on
GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

GROUP = 32


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int        # first global instance index of this rank
    count: int        # instances on this rank
    group_offset: int  # first global group (= first // 32)

    @property
    def groups(self) -> int:
        return (self.count + GROUP - 1) // GROUP


def shard_instances(n: int, world: int, rank: int) -> Shard:
    """Split [0, n) into `world` contiguous blocks of whole groups (sizes differ by <= 1 group)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    if n < 0:
        raise ValueError("n must be non-negative")
    total_groups = (n + GROUP - 1) // GROUP
    base, extra = divmod(total_groups, world)
    g0 = rank * base + min(rank, extra)
    g1 = g0 + base + (1 if rank < extra else 0)
    first = min(g0 * GROUP, n)
    last = min(g1 * GROUP, n)
    return Shard(rank, world, first, last - first, g0)


def to_i64(u: int) -> int:
    u &= (1 << 64) - 1
    return u - (1 << 64) if u >= (1 << 63) else u


def from_i64(i: int) -> int:
    return i & ((1 << 64) - 1)


def allreduce_checksum(local_sum: int, device=None, group=None) -> int:
    """Sum per-rank uint64 checksums mod 2^64 across the process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return from_i64(to_i64(local_sum))
    t = torch.tensor([to_i64(local_sum)], dtype=torch.int64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)  # two's-complement wrap == mod 2^64
    return from_i64(int(t.item()))


def counter_generator(key: bytes, n: int, world: int = 1, rank: int = 0, device: int = 0, first_index: int = 0):
    """A MickeyGenerator holding this rank's slice of the counter-IV set."""
    from .generator import MickeyGenerator

    sh = shard_instances(n, world, rank)
    gen = MickeyGenerator(device)
    gen.init_counter(key, first_index + sh.first, sh.count)
    gen.set_group_offset((first_index // GROUP) + sh.group_offset)
    return gen, sh
