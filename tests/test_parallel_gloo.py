"""World-size-2 gloo tests (CPU) of the N>1 host logic: token sharding + covariance SUM
all-reduce reproduces the unsharded accumulation; head/batch shards partition exactly;
max-over-ranks timing."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_17757_b200 import parallel as par


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle as O
        from paper_2605_17757_b200 import synth
        rng = np.random.default_rng(3)
        Q = synth.gen_queries(rng, 1001, 8, 2, 128)          # same seed on every rank
        lo, hi = par.token_shard(Q.shape[0], rank, world)
        acc = torch.from_numpy(O.cov_accumulate(Q[lo:hi], 2))
        par.allreduce_covariances(acc, world)
        full = O.cov_accumulate(Q, 2)
        err = float(np.abs(acc.numpy() - full).max() / np.abs(full).max())
        t = par.max_over_ranks(float(rank + 1) * 1.5, world)
        q.put((rank, err, t, (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_sharded_covariance_allreduce_matches_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][3] == (0, 501) and res[1][3] == (501, 1001)
    for rank, err, t, _ in res:
        assert err < 1e-13
        assert t == 3.0


def test_shard_partitions():
    for world in [1, 2, 4, 8]:
        seen_kv, seen_q = [], []
        for r in range(world):
            a, b, qa, qb = par.kv_head_shard(8, 64, r, world)
            seen_kv += list(range(a, b))
            seen_q += list(range(qa, qb))
            assert (qb - qa) == (b - a) * 8
        assert seen_kv == list(range(8)) and seen_q == list(range(64))
        toks = []
        for r in range(world):
            lo, hi = par.token_shard(524288 + 3, r, world)
            toks.append((lo, hi))
        assert toks[0][0] == 0 and toks[-1][1] == 524291
        assert all(toks[i][1] == toks[i + 1][0] for i in range(world - 1))
