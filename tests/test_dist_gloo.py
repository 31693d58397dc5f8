"""world_size-2 gloo test of the multi-GPU host logic on CPU.

Each rank takes its shard of a counter-IV instance range, produces that
shard's column-major keystream with the ORACLE (the checker stands in for the
GPU here: the GPU-vs-oracle equality is what tests/test_gpu_parity.py proves),
computes the shard checksum with the shard's global group offset, and the
ranks combine the 8-byte sums with one all-reduce.  The result must equal the
single-process checksum and the reference-derived golden value.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_04750_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, T, key_hex, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mickey_oracle as orc

        sh = sharding.shard_instances(n, world, rank)
        keys, ivs = orc.counter_material(bytes.fromhex(key_hex), sh.first, sh.count)
        col = orc.bulk_colmajor(keys, ivs, 80, T)
        local = orc.checksum_colmajor(col, sh.group_offset)
        total = sharding.allreduce_checksum(local)
        q.put((rank, sh.first, sh.count, local, total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,T", [(256, 1024), (96, 64)])
def test_two_rank_checksum_allreduce(golden, oracle, n, T):
    key_hex = golden["counter_iv"][0]["key"]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, T, key_hex, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(r[2] for r in res) == n and res[0][1] == 0 and res[1][1] == res[0][2]
    keys, ivs = oracle.counter_material(bytes.fromhex(key_hex), 0, n)
    want = oracle.checksum_colmajor(oracle.bulk_colmajor(keys, ivs, 80, T))
    assert all(r[4] == want for r in res)
    assert (res[0][3] + res[1][3]) % (1 << 64) == want
    for c in golden["counter_iv"]:
        if (c["first"], c["n"], c["nclocks"]) == (0, n, T):
            assert f"{want:x}" == c["u64_wrap_sum"]
