"""Multi-GPU readiness on one GPU: the path shards by KV head with no
collective, so a rank's sub-context — its KV-head slice of parallel.kv_head_shard with the
matching query heads, its own pool and its R_K / R_V shard — must reproduce the unsharded
context's pool bytes and outputs for those heads BIT FOR BIT.

quantize_append is per (token, head) and so is bit-exact under any split.  attend folds split
partials, and with automatic split sizing the split count depends on the number of heads in the
context (fp32 summation order); with a fixed split size (attend_pages_per_split) the split
structure of every (sequence, head) is the same in both and the outputs are bit-identical."""
import numpy as np
import pytest

from paper_2605_17757_b200 import parallel as par
from paper_2605_17757_b200 import synth

pytestmark = pytest.mark.gpu

HQ, HKV, D, P = 32, 8, 128, 64


def _ctx(hq, hkv, variant, pps):
    from paper_2605_17757_b200 import binding as B
    o = B.Oscar(B.Config(num_q_heads=hq, num_kv_heads=hkv, bits=2, group_size=64, page_size=P,
                         attend_pages_per_split=pps))
    o.set_variant(variant)
    return o


def _run(o, K, V, q, kn, vn, RK, RV, L, pt, decode):
    import torch
    B, hkv = len(L), K[0].shape[1]
    mp = pt.shape[1]
    pool = torch.zeros((B * mp, hkv, o.page_bytes()), dtype=torch.uint8, device="cuda")
    for b in range(B):
        pos = torch.arange(L[b] - (1 if decode else 0), device="cuda")
        slots = (pt[b, pos // P].long() * P + pos % P).contiguous()
        o.quantize_append(K[b][: len(pos)].contiguous(), V[b][: len(pos)].contiguous(), slots, RK, RV, pool)
    seq = torch.tensor(L, dtype=torch.int32, device="cuda")
    ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, q.shape[1], D), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, q.shape[1]), dtype=torch.float32, device="cuda")
    if decode:
        o.decode_step(q, kn, vn, pt, seq, pool, RK, RV, ws, out, lse)
    else:
        o.attend(q, pt, seq, pool, RK, RV, ws, out, lse)
    torch.cuda.synchronize()
    return pool, out, lse


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("decode", [False, True])
def test_kv_head_shards_reproduce_unsharded(world, variant, decode):
    import torch
    gen = torch.Generator(device="cuda").manual_seed(100 + world + 10 * variant)
    L = [700, 129, 1, 333]
    B = len(L)
    mp = (max(L) + P - 1) // P
    pt = torch.randperm(B * mp, generator=gen, device="cuda").to(torch.int32).reshape(B, mp).contiguous()
    K = [synth.torch_keys(gen, L[b], HKV, D, "cuda") for b in range(B)]
    V = [synth.torch_values(gen, L[b], HKV, D, "cuda") for b in range(B)]
    q = synth.torch_decode_q(gen, B, HQ, D, "cuda")
    kn = synth.torch_keys(gen, B, HKV, D, "cuda")
    vn = synth.torch_values(gen, B, HKV, D, "cuda")
    RK, RV = synth.torch_rotation(gen, HKV, D, "cuda"), synth.torch_rotation(gen, HKV, D, "cuda")
    full_pool, full_out, full_lse = _run(_ctx(HQ, HKV, variant, 4), K, V, q, kn, vn, RK, RV, L, pt, decode)
    for rank in range(world):
        kv_lo, kv_hi, q_lo, q_hi = par.kv_head_shard(HKV, HQ, rank, world)
        o = _ctx(q_hi - q_lo, kv_hi - kv_lo, variant, 4)
        pool, out, lse = _run(o, [k[:, kv_lo:kv_hi] for k in K], [v[:, kv_lo:kv_hi] for v in V],
                              q[:, q_lo:q_hi].contiguous(), kn[:, kv_lo:kv_hi].contiguous(),
                              vn[:, kv_lo:kv_hi].contiguous(), RK[kv_lo:kv_hi].contiguous(),
                              RV[kv_lo:kv_hi].contiguous(), L, pt, decode)
        assert torch.equal(pool, full_pool[:, kv_lo:kv_hi]), (rank, "pool bytes")
        assert torch.equal(out.view(torch.int32), full_out[:, q_lo:q_hi].view(torch.int32)), (rank, "output")
        assert torch.equal(lse.view(torch.int32), full_lse[:, q_lo:q_hi].view(torch.int32)), (rank, "lse")
