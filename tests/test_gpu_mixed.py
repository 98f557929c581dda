"""GPU parity of the mixed-precision cache (NEXT-1; §4, Alg. 1):
bf16 sink + recent window segment merged with the INT2 history, and a literal Alg. 1 decode
simulation with demotion of the oldest recent row.  Bars as test_gpu_parity.py (fp32 output
<= 2e-3 max-abs vs the fp64 oracle)."""
import numpy as np
import pytest

import oracle as O
from paper_2605_17757_b200 import synth

pytestmark = pytest.mark.gpu


def T(x, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def make(**kw):
    from paper_2605_17757_b200 import binding as B
    return B.Oscar(B.Config(**kw))


def _run_mixed(o, q, pt, L, pool, RK, RV, sk, sv, slen):
    import torch
    B, Hq, _ = q.shape
    ws = torch.empty(o.attend_workspace_bytes(B, pt.shape[1]), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, Hq), dtype=torch.float32, device="cuda")
    o.attend_mixed(T(q, torch.bfloat16), T(pt), T(np.asarray(L, np.int32)), T(pool), T(RK), T(RV),
                   T(sk, torch.bfloat16), T(sv, torch.bfloat16), T(np.asarray(slen, np.int32)), ws, out, lse)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), lse.cpu().numpy()


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("Hq,Hkv,bits,G,L,slen,cap", [
    (32, 8, 2, 64, [700, 0, 65], [320, 9, 0], 320),
    (4, 1, 4, 32, [130, 1], [1, 200], 256),
])
def test_attend_mixed_parity(variant, Hq, Hkv, bits, G, L, slen, cap):
    rng = np.random.default_rng(41 + Hq + cap)
    fmt = O.PageFormat(128, bits, G, 64)
    B = len(L)
    max_pages = max(1, (max(L) + 63) // 64)
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    pool = np.zeros((B * max_pages, Hkv, fmt.page_bytes), np.uint8)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    for b in range(B):
        if L[b]:
            slots = synth.slots_for(pt[b:b + 1], np.arange(L[b])[None], 64).reshape(-1)
            O.quantize_append(synth.gen_keys(rng, L[b], Hkv, 128), synth.gen_values(rng, L[b], Hkv, 128),
                              slots, RK, RV, fmt, pool)
    sk = synth.gen_keys(rng, B * Hkv * cap, 1, 128).reshape(B, Hkv, cap, 128)
    sv = synth.gen_values(rng, B * Hkv * cap, 1, 128).reshape(B, Hkv, cap, 128)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    ref, ref_lse = O.attend_mixed(q, pt, L, pool, sk, sv, slen, RK, RV, fmt, Hkv)
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=bits, group_size=G)
    o.set_variant(variant)
    got, lse = _run_mixed(o, q, pt, L, pool, RK, RV, sk, sv, slen)
    assert np.abs(got - ref).max() <= 2e-3
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isfinite(lse), fin)
    assert (np.abs(lse[fin] - ref_lse[fin]) <= 1e-3 + 1e-4 * np.abs(ref_lse[fin])).all()


def test_alg1_decode_simulation_with_demotion():
    """Alg. 1: prefill (sink raw, middle rotated+quantized, last W raw), then decode steps that
    append raw rows to the recent window and demote the oldest one once |recent| > W
    (P:L1614-1631), attending after each step.  The GPU path (quantize_append +
    attend_mixed) and the oracle path keep the same bookkeeping."""
    import torch
    rng = np.random.default_rng(77)
    B, Hq, Hkv, S0, W, L0, steps = 2, 8, 2, 4, 8, 40, 12
    fmt = O.PageFormat(128, 2, 64, 64)
    max_pages = 2
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64)
    gpool = torch.zeros((B * max_pages, Hkv, o.page_bytes()), dtype=torch.uint8, device="cuda")
    opool = np.zeros((B * max_pages, Hkv, fmt.page_bytes), np.uint8)
    cap = S0 + W + 1
    sk = np.zeros((B, Hkv, cap, 128), np.float32)
    sv = np.zeros((B, Hkv, cap, 128), np.float32)
    sink = [[] for _ in range(B)]
    recent = [[] for _ in range(B)]
    nhist = [0] * B

    def demote(b, k, v):
        slot = synth.slots_for(pt[b:b + 1], np.array([[nhist[b]]]), 64).reshape(-1)
        O.quantize_append(k[None], v[None], slot, RK, RV, fmt, opool)
        o.quantize_append(T(k[None], torch.bfloat16), T(v[None], torch.bfloat16), T(slot), T(RK), T(RV), gpool)
        nhist[b] += 1

    def push(b, k, v):
        if len(sink[b]) < S0:
            sink[b].append((k, v))
            return
        recent[b].append((k, v))
        if len(recent[b]) > W:
            kk, vv = recent[b].pop(0)
            demote(b, kk, vv)

    K0 = synth.gen_keys(rng, B * L0, Hkv, 128).reshape(B, L0, Hkv, 128)
    V0 = synth.gen_values(rng, B * L0, Hkv, 128).reshape(B, L0, Hkv, 128)
    for b in range(B):
        for t in range(L0):
            push(b, K0[b, t], V0[b, t])
    for step in range(steps):
        k = synth.gen_keys(rng, B, Hkv, 128)
        v = synth.gen_values(rng, B, Hkv, 128)
        for b in range(B):
            push(b, k[b], v[b])
        seglen = []
        for b in range(B):
            rows = sink[b] + recent[b]
            for j, (kk, vv) in enumerate(rows):
                sk[b, :, j] = kk
                sv[b, :, j] = vv
            seglen.append(len(rows))
            assert len(sink[b]) + len(recent[b]) + nhist[b] == L0 + step + 1      # partition
        q = synth.gen_decode_q(rng, B, Hq, 128)
        ref, _ = O.attend_mixed(q, pt, nhist, opool, sk, sv, seglen, RK, RV, fmt, Hkv)
        got, _ = _run_mixed(o, q, pt, nhist, gpool.cpu().numpy(), RK, RV, sk, sv, seglen)
        assert np.abs(got - ref).max() <= 2e-3, step
