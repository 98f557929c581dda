"""GPU parity of oscar_decode_step — one Alg. 1 DecodeStep: QuantizeAndWrite of
the step's new K/V row at position seq_lens[b]-1, then attention over the
seq_lens[b] tokens including it (reading Z20).  The oracle runs the same two steps with its own
quantize_append and attend on the same seeded inputs.  Bars as test_gpu_parity.py: pool bytes
equal except rounding-boundary flips of the fp32 rotation, outputs within 2e-3 max-abs (fp32
output mode), lse within the IMMA path's 15-bit q̃ bound."""
import zlib

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


def check_step_pool(got_pool, ref_pool, pt, L, k_new, v_new, RK, RV, fmt, live, seqs=None):
    """The history (first L-1 tokens of each sequence) is untouched, and the step's new rows equal
    the oracle's up to validated rounding-boundary flips (oracle/boundary.py)."""
    from oracle.boundary import check_pool_flips
    Hkv = RK.shape[0]
    for b in (range(len(L)) if seqs is None else seqs):
        hist = synth.slots_for(pt[b:b + 1], np.arange(max(L[b] - 1, 0))[None], fmt.P).reshape(-1)
        for h in range(Hkv):
            a, r = O.read_codes(got_pool, hist, h, fmt), O.read_codes(ref_pool, hist, h, fmt)
            assert all(np.array_equal(x.view(np.uint8), y.view(np.uint8)) for x, y in zip(a, r))
    lv = [b for b in live if seqs is None or b in seqs]
    if lv:
        ns = np.array([pt[b, (L[b] - 1) // fmt.P] * fmt.P + (L[b] - 1) % fmt.P for b in lv], np.int64)
        check_pool_flips(got_pool, {"K": O.rotate(k_new[lv], RK), "V": O.rotate(v_new[lv], RV)}, ns, fmt)


@pytest.mark.parametrize("cfg", [
    dict(name="C2small", Hq=32, Hkv=8, bits=2, G=64, L=[1000, 65, 1, 64, 129]),   # new page, 1-token seq
    dict(name="g8", Hq=16, Hkv=2, bits=2, G=64, L=[700, 130]),
    dict(name="b4G32", Hq=8, Hkv=2, bits=4, G=32, L=[450, 64]),
    dict(name="g1", Hq=2, Hkv=2, bits=2, G=128, L=[300]),
    dict(name="b3", Hq=8, Hkv=2, bits=3, G=64, L=[333, 2]),                        # simple kernels
    dict(name="empty", Hq=8, Hkv=2, bits=2, G=64, L=[200, 0]),                     # seq_len 0: no append
])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("prerot_v", [False, True])
def test_decode_step_parity(cfg, variant, prerot_v):
    import torch
    rng = np.random.default_rng(zlib.crc32(f"{cfg['name']}/{variant}/{prerot_v}".encode()))
    Hq, Hkv, L = cfg["Hq"], cfg["Hkv"], cfg["L"]
    B = len(L)
    fmt = O.PageFormat(128, cfg["bits"], cfg["G"], 64)
    max_pages = max(1, (max(L) + 63) // 64)
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    RK = synth.gen_rotation(rng, Hkv, 128)
    RV = np.broadcast_to(np.eye(128, dtype=np.float32), (Hkv, 128, 128)).copy() if prerot_v \
        else synth.gen_rotation(rng, Hkv, 128)
    pool = np.zeros((B * max_pages, Hkv, fmt.page_bytes), np.uint8)
    for b in range(B):                       # history: the first L-1 tokens, written by the oracle
        n = max(L[b] - 1, 0)
        if n:
            slots = synth.slots_for(pt[b:b + 1], np.arange(n)[None], 64).reshape(-1)
            O.quantize_append(synth.gen_keys(rng, n, Hkv, 128), synth.gen_values(rng, n, Hkv, 128), slots,
                              RK, RV, fmt, pool)
    k_new = synth.gen_keys(rng, B, Hkv, 128)
    v_new = synth.gen_values(rng, B, Hkv, 128)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    # oracle: QuantizeAndWrite at position L-1, then attend over L tokens
    ref_pool = pool.copy()
    live = [b for b in range(B) if L[b] > 0]
    new_slots = np.array([pt[b, (L[b] - 1) // 64] * 64 + (L[b] - 1) % 64 for b in live], np.int64)
    O.quantize_append(k_new[live], v_new[live], new_slots, RK, RV, fmt, ref_pool)
    ref, ref_lse = O.attend(q, pt, L, ref_pool, RK, RV, fmt, Hkv)

    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=cfg["bits"], group_size=cfg["G"])
    o.set_variant(variant)
    gpool = T(pool)
    ws = torch.empty(o.attend_workspace_bytes(B, max_pages), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, Hq), dtype=torch.float32, device="cuda")
    o.decode_step(T(q, torch.bfloat16), T(k_new, torch.bfloat16), T(v_new, torch.bfloat16), T(pt),
                  T(np.asarray(L, np.int32)), gpool, T(RK), None if prerot_v else T(RV), ws, out, lse)
    torch.cuda.synchronize()
    got_pool = gpool.cpu().numpy()
    check_step_pool(got_pool, ref_pool, pt, L, k_new, v_new, RK, RV, fmt, live)
    assert np.abs(out.cpu().numpy() - ref).max() <= 2e-3
    lg = lse.cpu().numpy()
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isfinite(lg), fin)
    assert (np.abs(lg[fin] - ref_lse[fin]) <= 1e-3 + 1e-4 * np.abs(ref_lse[fin])).all()


def test_decode_step_equals_append_then_attend():
    """The fused call and the two-call sequence (quantize_append, then attend) agree."""
    import torch
    rng = np.random.default_rng(11)
    Hq, Hkv, B, L = 32, 8, 4, [640, 1000, 64, 65]
    fmt = O.PageFormat(128, 2, 64, 64)
    max_pages = (max(L) + 63) // 64
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    pool = np.zeros((B * max_pages, Hkv, fmt.page_bytes), np.uint8)
    for b in range(B):
        n = L[b] - 1
        slots = synth.slots_for(pt[b:b + 1], np.arange(n)[None], 64).reshape(-1)
        O.quantize_append(synth.gen_keys(rng, n, Hkv, 128), synth.gen_values(rng, n, Hkv, 128), slots, RK, RV,
                          fmt, pool)
    k_new, v_new = synth.gen_keys(rng, B, Hkv, 128), synth.gen_values(rng, B, Hkv, 128)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    o = make(num_q_heads=Hq, num_kv_heads=Hkv)
    ws = torch.empty(o.attend_workspace_bytes(B, max_pages), dtype=torch.uint8, device="cuda")
    args = (T(pt), T(np.asarray(L, np.int32)))
    p1, p2 = T(pool), T(pool)
    o1 = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    o2 = torch.empty_like(o1)
    o.decode_step(T(q, torch.bfloat16), T(k_new, torch.bfloat16), T(v_new, torch.bfloat16), *args, p1, T(RK),
                  T(RV), ws, o1)
    slots = T(np.array([pt[b, (L[b] - 1) // 64] * 64 + (L[b] - 1) % 64 for b in range(B)], np.int64))
    o.quantize_append(T(k_new, torch.bfloat16), T(v_new, torch.bfloat16), slots, T(RK), T(RV), p2)
    o.attend(T(q, torch.bfloat16), *args, p2, T(RK), T(RV), ws, o2)
    torch.cuda.synchronize()
    for p_ in (p1, p2):                      # both pools: oracle up to validated boundary flips
        check_step_pool(p_.cpu().numpy(), pool_ref_after(pool, pt, L, k_new, v_new, RK, RV, fmt), pt, L,
                        k_new, v_new, RK, RV, fmt, list(range(B)))
    # the fused step folds the new token as its own partial (fp32 logit q̃·k̂), the two-call path
    # through the IMMA kernel (15-bit q̃, reading Z31): equal up to that rounding
    assert (o1 - o2).abs().max().item() <= (2e-4 if torch.equal(p1, p2) else 2e-3)


def pool_ref_after(pool, pt, L, k_new, v_new, RK, RV, fmt):
    ref = pool.copy()
    live = [b for b in range(len(L)) if L[b] > 0]
    ns = np.array([pt[b, (L[b] - 1) // fmt.P] * fmt.P + (L[b] - 1) % fmt.P for b in live], np.int64)
    O.quantize_append(k_new[live], v_new[live], ns, RK, RV, fmt, ref)
    return ref


def test_decode_step_full_size_c2():
    """oscar_decode_step at the bench's C2 launch configuration (B = 16, L = 32768, 32 q / 8 kv
    heads, 2-bit, G = 64; one sequence ragged), on a seeded random packed history: the step's new
    rows are checked for all 16 sequences (validated boundary flips only), the history of the
    sampled sequences is untouched, and the outputs of two sequences (all 32 heads) match the
    oracle run on the same history plus its own QuantizeAndWrite of the new rows."""
    import torch
    B, L0, Hq, Hkv, P = 16, 32768, 32, 8, 64
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64)
    fmt = O.PageFormat(128, 2, 64, P)
    max_pages = L0 // P
    gen = torch.Generator(device="cuda").manual_seed(3)
    pool = synth.torch_random_pool(gen, B * max_pages, Hkv, o.page_bytes(), fmt.meta_off, P * 2, "cuda")
    rng = np.random.default_rng(3)
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    kn, vn = synth.gen_keys(rng, B, Hkv, 128), synth.gen_values(rng, B, Hkv, 128)
    L = [L0] * B
    L[9] = L0 - 777
    sample = [0, 9]
    host_before = {b: pool[torch.from_numpy(pt[b].astype(np.int64)).cuda()].cpu().numpy() for b in sample}
    ws = torch.empty(o.attend_workspace_bytes(B, max_pages), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    o.decode_step(T(q, torch.bfloat16), T(kn, torch.bfloat16), T(vn, torch.bfloat16), T(pt),
                  T(np.asarray(L, np.int32)), pool, T(RK), T(RV), ws, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    # new rows of all 16 sequences: pages holding position L-1
    newp = np.array([pt[b, (L[b] - 1) // P] for b in range(B)], np.int64)
    sub = pool[torch.from_numpy(newp).cuda()].cpu().numpy()          # [B pages, Hkv, bytes]
    from oracle.boundary import check_pool_flips
    ns = np.array([b * P + (L[b] - 1) % P for b in range(B)], np.int64)
    check_pool_flips(sub, {"K": O.rotate(kn, RK), "V": O.rotate(vn, RV)}, ns, fmt)
    for b in sample:
        loc = np.arange(max_pages, dtype=np.int32)[None]
        after = pool[torch.from_numpy(pt[b].astype(np.int64)).cuda()].cpu().numpy()
        ref_pool = host_before[b].copy()
        O.quantize_append(kn[b:b + 1], vn[b:b + 1], np.array([L[b] - 1], np.int64), RK, RV, fmt, ref_pool)
        hist = np.arange(L[b] - 1)
        for h in range(Hkv):                 # the history the partial kernel read is untouched
            a, r = O.read_codes(after, hist[::97], h, fmt), O.read_codes(ref_pool, hist[::97], h, fmt)
            assert all(np.array_equal(x.view(np.uint8), y.view(np.uint8)) for x, y in zip(a, r))
        ref, _ = O.attend(q[b:b + 1], loc, [L[b]], ref_pool, RK, RV, fmt, Hkv)
        assert np.abs(got[b] - ref[0]).max() <= 2e-3
