"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Tolerances (north star):
  * rotated values: per row max|Δ| / ‖x̃‖₂ <= 1e-5                     (reading Z26)
  * codes / metadata / pool bytes: bit-exact given identical rotated inputs
  * full append: bit-exact except rounding-boundary flips, every one validated
    (oracle/boundary.py: |Δcode| = 1 with the oracle's pre-round value within the 1e-5 rotation
    bound of .5, or fp16 metadata one ulp apart at a rounding midpoint)
  * attention: fp32-output mode <= 2e-3 max-abs vs the fp64 oracle; bf16 mode ==
    RNE(fp32 mode) bit-for-bit (reading Z25)
"""
import math
import zlib

import numpy as np
import pytest

import oracle as O
from paper_2605_17757_b200 import synth

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def T(x, dtype=None):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def make(**kw):
    from paper_2605_17757_b200 import binding as B
    return B.Oscar(B.Config(**kw))


ALL_BG = [(b, g) for b in (2, 3, 4) for g in (32, 64, 128)]


# ---------------------------------------------------------------------------- rotation
# oscar_rotate takes the route oscar_quantize_append takes for the same T and config (api.cu
# append_path): T <= 64 -> append_small_kernel, else the tcgen05 append_tc_kernel (MODE 1: its
# TMEM rows dumped as fp32), variant 1 -> the simple kernel.  Every <b, G> instance of the
# tensor-core kernel is checked (the rotation is shared, the instances differ in the epilogue).
@pytest.mark.parametrize("bits,G", ALL_BG)
@pytest.mark.parametrize("T_", [33, 300])
@pytest.mark.parametrize("variant", [0, 1])
def test_rotate_parity(bits, G, T_, variant):
    torch = _torch()
    rng = np.random.default_rng(100 + T_ + bits * 7 + G)
    H = 3
    X = synth.gen_keys(rng, T_, H, 128)
    R = synth.gen_rotation(rng, H, 128)
    o = make(num_q_heads=H, num_kv_heads=H, bits=bits, group_size=G)
    o.set_variant(variant)
    out = torch.full((T_, H, 128), float("nan"), dtype=torch.float32, device="cuda")
    o.rotate(T(X, torch.bfloat16), T(R), out)
    ref = O.rotate(X, R).astype(np.float64)
    got = out.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max(axis=-1) / np.linalg.norm(ref, axis=-1)
    assert err.max() <= 1e-5, err.max()


@pytest.mark.parametrize("T_", [1, 129, 1000])
def test_rotate_fwht_parity(T_):
    """oscar_rotate_fwht (the U-GEMM + Walsh–Hadamard form of the rotation, measured against the
    dense form in DESIGN.md §7.2): ((x·U)·H)·P_br against the oracle's x·compose_rotation(U),
    per row <= 1e-5 of ||x̃|| (reading Z26)."""
    torch = _torch()
    rng = np.random.default_rng(300 + T_)
    H = 2
    X = synth.gen_keys(rng, T_, H, 128)
    U = np.stack([np.linalg.qr(rng.standard_normal((128, 128)))[0] for _ in range(H)]).astype(np.float32)
    R = np.stack([O.compose_rotation(U[h].astype(np.float64)) for h in range(H)]).astype(np.float32)
    o = make(num_q_heads=H, num_kv_heads=H, bits=2, group_size=64)
    out = torch.full((T_, H, 128), float("nan"), dtype=torch.float32, device="cuda")
    o.rotate_fwht(T(X, torch.bfloat16), T(U), out)
    ref = O.rotate(X, R).astype(np.float64)
    got = out.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max(axis=-1) / np.linalg.norm(ref, axis=-1)
    assert err.max() <= 1e-5, err.max()


# ---------------------------------------------------------------------------- quantizer
def _adversarial_rows(rng, n, H):
    X = rng.standard_normal((n, H, 128)).astype(np.float32) * rng.uniform(0.01, 30, (n, H, 1)).astype(np.float32)
    X[0] = 0.0                                       # zero rows: s16 = 0
    X[1, :, :64] = 3.25                              # constant group
    X[2] *= 1e-7                                     # s underflows fp16 -> s16 = 0 / subnormal
    X[3] = np.round(X[3] * 2) / 2                    # many exact half-steps
    X[4, :, ::2] = 7.0; X[4, :, 1::2] = -7.0         # two-valued groups
    return X


# oscar_quantize_rotated ("identical rotated inputs"): the route of quantize_append for that T —
# T = 333: the tcgen05 kernel's epilogue (MODE 2, no clipping) / the simple kernel (clipping,
# variant 1); T = 40: append_small_kernel's epilogue.  Bit-exact pool bytes.
@pytest.mark.parametrize("bits,G,rho", [(b, g, (1.0, 1.0)) for b, g in ALL_BG] + [
    (2, 32, (0.96, 0.92)), (4, 128, (0.96, 0.92)), (2, 128, (0.5, 0.999)), (3, 64, (0.96, 0.92))])
@pytest.mark.parametrize("Tn", [333, 40])
@pytest.mark.parametrize("variant", [0, 1])
def test_quantize_rotated_bit_exact(bits, G, rho, Tn, variant):
    torch = _torch()
    rng = np.random.default_rng(bits * 1000 + G + Tn)
    H, npages = 2, 8
    fmt = O.PageFormat(128, bits, G, 64)
    Kr = _adversarial_rows(rng, Tn, H)
    Vr = _adversarial_rows(rng, Tn, H)[::-1].copy()
    slots = rng.permutation(npages * 64)[:Tn].astype(np.int64)
    if Tn == 333:                                    # a 16-aligned run: the staged-V 16-B store path
        slots[100:164] = np.arange(320, 384)
        rest = np.setdiff1d(np.arange(npages * 64), slots[100:164])
        others = np.concatenate([np.arange(100), np.arange(164, Tn)])
        slots[others] = rng.permutation(rest)[:len(others)]
    ref = np.zeros((npages, H, fmt.page_bytes), np.uint8)
    O.quantize_rotated(Kr, Vr, slots, fmt, ref, rho[0], rho[1])
    o = make(num_q_heads=H, num_kv_heads=H, bits=bits, group_size=G, clip_ratio_k=rho[0],
             clip_ratio_v=rho[1])
    o.set_variant(variant)
    pool = torch.zeros((npages, H, o.page_bytes()), dtype=torch.uint8, device="cuda")
    o.quantize_rotated(T(Kr), T(Vr), T(slots), pool)
    got = pool.cpu().numpy()
    diff = np.argwhere(got != ref)
    assert diff.size == 0, f"{len(diff)} bytes differ, first {diff[:5]}"


# ---------------------------------------------------------------------------- full append
def _slots(rng, mode, Tn, npages):
    """perm: random distinct slots.  contigN: the first 700 tokens take consecutive slots from
    slot N (a 16-aligned N exercises the tensor-core kernel's staged V path, also across page
    boundaries), the rest random distinct slots."""
    if mode == "perm":
        return rng.permutation(npages * 64)[:Tn].astype(np.int64)
    start = int(mode[6:])
    run = np.arange(start, start + min(700, Tn))
    rest = np.setdiff1d(np.arange(npages * 64), run)
    return np.concatenate([run, rng.permutation(rest)[:Tn - len(run)]]).astype(np.int64)


def check_append_flips(got, K, V, RK, RV, slots, fmt, rho=(1.0, 1.0)):
    """Every byte that differs from the oracle's pool must be a rounding-boundary flip of the
    fp32 rotation (oracle/boundary.py: codes |Δ| = 1 with the oracle's pre-round value within the
    1e-5 rotation bound of .5, or fp16 metadata one ulp apart at a rounding midpoint)."""
    from oracle.boundary import check_pool_flips
    rot = {"K": O.rotate(K, RK), "V": O.rotate(V, RV)}
    return check_pool_flips(got, rot, slots, fmt, rho)


@pytest.mark.parametrize("bits,G,rho,variant,Tn,slot_mode", [
    (2, 64, (1.0, 1.0), 0, 1000, "perm"), (4, 32, (0.96, 0.92), 0, 1000, "perm"),
    (2, 64, (1.0, 1.0), 1, 1000, "perm"), (2, 32, (1.0, 1.0), 0, 16, "perm"),
    (4, 64, (1.0, 1.0), 0, 300, "perm"), (4, 32, (1.0, 1.0), 0, 1280, "perm"),
    (2, 128, (1.0, 1.0), 0, 129, "perm"),
    (2, 64, (1.0, 1.0), 0, 1000, "contig208"), (4, 64, (1.0, 1.0), 0, 1000, "contig208"),
    (3, 64, (1.0, 1.0), 0, 1000, "perm"), (3, 32, (0.96, 0.92), 0, 300, "contig208"),
    (3, 128, (1.0, 1.0), 0, 40, "perm"),
    (2, 32, (1.0, 1.0), 0, 1000, "contig200"), (4, 32, (1.0, 1.0), 0, 1280, "contig0"),
    (2, 128, (1.0, 1.0), 0, 1000, "contig208"), (4, 128, (1.0, 1.0), 0, 1000, "perm"),   # G = 128 on tcgen05
    (3, 64, (1.0, 1.0), 0, 1000, "contig208"), (3, 128, (1.0, 1.0), 0, 1000, "perm"),    # 3-bit on tcgen05
    (3, 32, (1.0, 1.0), 0, 1000, "contig200"),
])
def test_quantize_append_parity(bits, G, rho, variant, Tn, slot_mode):
    torch = _torch()
    rng = np.random.default_rng(7 + bits + G + Tn)
    H, npages = 8, 21
    fmt = O.PageFormat(128, bits, G, 64)
    K = synth.gen_keys(rng, Tn, H, 128)
    V = synth.gen_values(rng, Tn, H, 128)
    RK, RV = synth.gen_rotation(rng, H, 128), synth.gen_rotation(rng, H, 128)
    slots = _slots(rng, slot_mode, Tn, npages)
    ref = np.zeros((npages, H, fmt.page_bytes), np.uint8)
    O.quantize_append(K, V, slots, RK, RV, fmt, ref, rho[0], rho[1])
    o = make(num_q_heads=H * 4, num_kv_heads=H, bits=bits, group_size=G, clip_ratio_k=rho[0],
             clip_ratio_v=rho[1])
    o.set_variant(variant)
    pool = torch.zeros((npages, H, o.page_bytes()), dtype=torch.uint8, device="cuda")
    o.quantize_append(T(K, torch.bfloat16), T(V, torch.bfloat16), T(slots), T(RK), T(RV), pool)
    got = pool.cpu().numpy()
    # every written byte equals the oracle's up to validated boundary flips; untouched slots stay 0
    st = check_append_flips(got, K, V, RK, RV, slots, fmt, rho)
    free = np.setdiff1d(np.arange(npages * 64), slots)
    for h in range(H):
        ck, cv, m = O.read_codes(got, free, h, fmt)
        assert not ck.any() and not cv.any() and not m.view(np.uint16).any()
    assert st["code_flips"] + st["meta_flips"] <= 1e-3 * st["groups"] * G, st


@pytest.mark.parametrize("P,bits,G", [(16, 2, 64), (256, 2, 128), (32, 4, 32), (128, 4, 64), (48, 3, 32)])
def test_quantize_append_page_sizes(P, bits, G):
    """Other page sizes through the default (tensor-core where supported) append: 700 tokens in
    consecutive slots from a 16-aligned start (staged V path) plus random slots."""
    torch = _torch()
    rng = np.random.default_rng(P + bits * 10 + G)
    H, Tn = 4, 1000
    npages = (2000 + P - 1) // P
    fmt = O.PageFormat(128, bits, G, P)
    K, V = synth.gen_keys(rng, Tn, H, 128), synth.gen_values(rng, Tn, H, 128)
    RK, RV = synth.gen_rotation(rng, H, 128), synth.gen_rotation(rng, H, 128)
    run = np.arange(208, 908)
    rest = np.setdiff1d(np.arange(npages * P), run)
    slots = np.concatenate([run, rng.permutation(rest)[:Tn - 700]]).astype(np.int64)
    ref = np.zeros((npages, H, fmt.page_bytes), np.uint8)
    O.quantize_append(K, V, slots, RK, RV, fmt, ref)
    o = make(num_q_heads=H * 4, num_kv_heads=H, bits=bits, group_size=G, page_size=P)
    pool = torch.zeros((npages, H, o.page_bytes()), dtype=torch.uint8, device="cuda")
    o.quantize_append(T(K, torch.bfloat16), T(V, torch.bfloat16), T(slots), T(RK), T(RV), pool)
    check_append_flips(pool.cpu().numpy(), K, V, RK, RV, slots, fmt)


def test_quantize_append_misaligned_falls_back():
    """Row bases that are not 16-B aligned (TMA cannot take them) route to the simple kernel
    instead of failing; the result is the same pool up to boundary flips."""
    torch = _torch()
    rng = np.random.default_rng(77)
    H, Tn, npages = 2, 300, 8
    fmt = O.PageFormat(128, 2, 64, 64)
    K, V = synth.gen_keys(rng, Tn, H, 128), synth.gen_values(rng, Tn, H, 128)
    RK, RV = synth.gen_rotation(rng, H, 128), synth.gen_rotation(rng, H, 128)
    slots = rng.permutation(npages * 64)[:Tn].astype(np.int64)
    o = make(num_q_heads=H, num_kv_heads=H)
    kb = torch.zeros(Tn * H * 128 + 1, dtype=torch.bfloat16, device="cuda")
    vb = torch.zeros_like(kb)
    kb[1:] = T(K, torch.bfloat16).reshape(-1)
    vb[1:] = T(V, torch.bfloat16).reshape(-1)
    Km, Vm = kb[1:].view(Tn, H, 128), vb[1:].view(Tn, H, 128)     # 2-byte offset: misaligned
    pool = torch.zeros((npages, H, o.page_bytes()), dtype=torch.uint8, device="cuda")
    o.quantize_append(Km, Vm, T(slots), T(RK), T(RV), pool)
    check_append_flips(pool.cpu().numpy(), K, V, RK, RV, slots, fmt)


# ---------------------------------------------------------------------------- attention
def _oracle_pool(rng, fmt, B, Hkv, L, shuffle=True):
    max_pages = (max(L) + fmt.P - 1) // fmt.P if len(L) else 1
    max_pages = max(max_pages, 1)
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng if shuffle else None)
    pool = np.zeros((B * max_pages, Hkv, fmt.page_bytes), np.uint8)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    for b in range(B):
        if L[b] == 0:
            continue
        K = synth.gen_keys(rng, L[b], Hkv, 128)
        V = synth.gen_values(rng, L[b], Hkv, 128)
        slots = synth.slots_for(pt[b:b + 1], np.arange(L[b])[None], fmt.P).reshape(-1)
        O.quantize_append(K, V, slots, RK, RV, fmt, pool)
    return pt, pool, RK, RV


def _run_attend(o, q, pt, L, pool, RK, RV):
    torch = _torch()
    B, Hq, _ = q.shape
    ws = torch.empty(o.attend_workspace_bytes(B, pt.shape[1]), dtype=torch.uint8, device="cuda")
    out32 = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    out16 = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((B, Hq), dtype=torch.float32, device="cuda")
    args = (T(q, torch.bfloat16), T(pt), T(np.asarray(L, np.int32)), T(pool), T(RK), T(RV), ws)
    o.attend(*args, out32, lse)
    o.attend(*args, out16)
    torch.cuda.synchronize()
    return out32, out16, lse


def _z31_lse_bound(q, pt, L, pool, RK, fmt, Hkv):
    """Reading Z31: the tensor-core path rounds q̃ = q·R_K·scale·log2(e) to integers of step
    qscale = max|q̃| / 32639, so every logit (log2 units) moves by at most (qscale / 2)·‖k̂_t‖₁
    and so does log2 Σ 2^logit; in natural-log units x ln 2.  Per (sequence, query head)."""
    B, Hq, d = q.shape
    g = Hq // Hkv
    out = np.zeros((B, Hq))
    for b in range(B):
        if L[b] == 0:
            continue
        slots = np.asarray(pt[b], np.int64)[np.arange(L[b]) // fmt.P] * fmt.P + np.arange(L[b]) % fmt.P
        for h in range(Hkv):
            Kh, _ = O.read_rows(pool, slots, h, fmt)
            k1 = np.abs(Kh).sum(axis=1).max()
            for i in range(h * g, (h + 1) * g):
                qt = np.asarray(q[b, i], np.float64) @ RK[h] / math.sqrt(d) * math.log2(math.e)
                out[b, i] = math.log(2) * 0.5 * np.abs(qt).max() / 32639 * k1
    return out


@pytest.mark.parametrize("cfg", [
    dict(name="C1", Hq=1, Hkv=1, bits=4, G=32, B=64, L="ramp256"),
    dict(name="C2small", Hq=32, Hkv=8, bits=2, G=64, B=3, L=[1000, 77, 0]),
    dict(name="g8", Hq=16, Hkv=2, bits=2, G=128, B=2, L=[513, 64]),
    dict(name="g2b4", Hq=4, Hkv=2, bits=4, G=64, B=2, L=[300, 1]),
    dict(name="C4small", Hq=16, Hkv=2, bits=2, G=64, B=2, L=[700, 130]),     # g=8, two 8-combo tiles
    dict(name="g4G32", Hq=8, Hkv=2, bits=4, G=32, B=2, L=[450, 64]),        # 4 groups x 4 heads
    dict(name="b3", Hq=8, Hkv=2, bits=3, G=64, B=2, L=[333, 64]),           # 3-bit: simple kernels
    dict(name="C2G32", Hq=32, Hkv=8, bits=2, G=32, B=3, L=[1000, 77, 0]),   # token-row layout, 4 groups
    dict(name="b3G32", Hq=8, Hkv=2, bits=3, G=32, B=2, L=[290, 17]),
    dict(name="b3G128", Hq=16, Hkv=2, bits=3, G=128, B=2, L=[300, 64]),
    dict(name="b4g8", Hq=16, Hkv=2, bits=4, G=64, B=2, L=[250, 1]),
    dict(name="b3g8G64", Hq=16, Hkv=2, bits=3, G=64, B=2, L=[400, 70]),    # 3-bit, group-pure PV tiles
    dict(name="b3C2", Hq=32, Hkv=8, bits=3, G=64, B=3, L=[1000, 77, 0]),   # 3-bit token-row layout
])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("pps", [0, 1, 3])
@pytest.mark.parametrize("qsig", [2.0, 8.0])          # 8.0: the "peaky" decode q
def test_attend_parity(cfg, variant, pps, qsig):
    torch = _torch()
    rng = np.random.default_rng(zlib.crc32(cfg["name"].encode()))    # stable across processes
    fmt = O.PageFormat(128, cfg["bits"], cfg["G"], 64)
    L = list(range(4, 260, 4)) if cfg["L"] == "ramp256" else cfg["L"]
    B = cfg["B"]
    pt, pool, RK, RV = _oracle_pool(rng, fmt, B, cfg["Hkv"], L)
    q = synth.gen_decode_q(rng, B, cfg["Hq"], 128, sigma=qsig)
    ref, ref_lse = O.attend(q, pt, L, pool, RK, RV, fmt, cfg["Hkv"])
    o = make(num_q_heads=cfg["Hq"], num_kv_heads=cfg["Hkv"], bits=cfg["bits"], group_size=cfg["G"],
             attend_pages_per_split=pps)
    o.set_variant(variant)
    out32, out16, lse = _run_attend(o, q, pt, L, pool, RK, RV)
    got = out32.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max()
    assert err <= 2e-3, err
    assert torch.equal(out32.to(torch.bfloat16).view(torch.int16), out16.view(torch.int16))
    lg = lse.cpu().numpy()
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isfinite(lg), fin)
    # lse: the IMMA path quantizes q̃ to 15 bits (reading Z31); the bound of that reading per row
    bound = _z31_lse_bound(q, pt, L, pool, RK, fmt, cfg["Hkv"]) + 1e-4 * np.abs(ref_lse) + 1e-4
    assert (np.abs(lg[fin] - ref_lse[fin]) <= bound[fin]).all()


@pytest.mark.parametrize("P,bits,G,Hq,Hkv", [(32, 2, 64, 32, 8), (128, 2, 64, 32, 8), (16, 2, 128, 16, 2),
                                            (256, 4, 64, 8, 2), (32, 4, 32, 8, 2), (48, 2, 64, 32, 8),
                                            (48, 3, 64, 8, 2), (256, 3, 128, 8, 2), (80, 3, 32, 4, 1)])
@pytest.mark.parametrize("variant", [0, 1])
def test_attend_page_sizes(P, bits, G, Hq, Hkv, variant):
    """Page sizes other than 64 (the FULL-page fast path never applies): tensor-core kernels'
    generic masked path against the oracle, ragged lengths; P that does not divide 128 takes the
    simple kernel's one-(token, head)-per-thread scoring path."""
    torch = _torch()
    rng = np.random.default_rng(P * 7 + bits + G)
    fmt = O.PageFormat(128, bits, G, P)
    L = [5 * P + 3, P, 1]
    pt, pool, RK, RV = _oracle_pool(rng, fmt, len(L), Hkv, L)
    q = synth.gen_decode_q(rng, len(L), Hq, 128)
    ref, _ = O.attend(q, pt, L, pool, RK, RV, fmt, Hkv)
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=bits, group_size=G, page_size=P)
    o.set_variant(variant)
    out32, out16, _ = _run_attend(o, q, pt, L, pool, RK, RV)
    assert np.abs(out32.cpu().numpy().astype(np.float64) - ref).max() <= 2e-3


@pytest.mark.parametrize("B,Hq,Hkv", [(1, 1, 1), (3, 1, 1), (1, 2, 1), (2, 1, 1), (3, 2, 2), (5, 4, 4)])
@pytest.mark.parametrize("call", ["attend", "decode_step", "attend_mixed"])
def test_attend_odd_row_counts(B, Hq, Hkv, call):
    """B·H_q odd or ≡ 2 mod 4 (the workspace sub-buffers must stay aligned for the
    prologue's 8-B and the segment kernel's 16-B stores): every entry point against the oracle."""
    torch = _torch()
    rng = np.random.default_rng(1000 * B + 10 * Hq + Hkv)
    fmt = O.PageFormat(128, 2, 64, 64)
    L = [int(x) for x in rng.integers(1, 200, B)]
    pt, pool, RK, RV = _oracle_pool(rng, fmt, B, Hkv, L)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64)
    mp = pt.shape[1]
    ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    if call == "attend":
        o.attend(T(q, torch.bfloat16), T(pt), T(np.asarray(L, np.int32)), T(pool), T(RK), T(RV), ws, out)
        ref, _ = O.attend(q, pt, L, pool, RK, RV, fmt, Hkv)
    elif call == "decode_step":
        kn, vn = synth.gen_keys(rng, B, Hkv, 128), synth.gen_values(rng, B, Hkv, 128)
        L1 = [x + 1 for x in L]
        mp1 = (max(L1) + 63) // 64
        if mp1 > mp:                                 # room for the new row
            pt = np.concatenate([pt, np.arange(pool.shape[0], pool.shape[0] + B, dtype=np.int32)[:, None]], 1)
            pool = np.concatenate([pool, np.zeros((B, Hkv, fmt.page_bytes), np.uint8)])
            ws = torch.empty(o.attend_workspace_bytes(B, pt.shape[1]), dtype=torch.uint8, device="cuda")
        ref_pool = pool.copy()
        ns = np.array([pt[b, (L1[b] - 1) // 64] * 64 + (L1[b] - 1) % 64 for b in range(B)], np.int64)
        O.quantize_append(kn, vn, ns, RK, RV, fmt, ref_pool)
        ref, _ = O.attend(q, pt, L1, ref_pool, RK, RV, fmt, Hkv)
        gp = T(pool)
        o.decode_step(T(q, torch.bfloat16), T(kn, torch.bfloat16), T(vn, torch.bfloat16), T(pt),
                      T(np.asarray(L1, np.int32)), gp, T(RK), T(RV), ws, out)
    else:
        cap = 8
        sk = synth.gen_keys(rng, B * Hkv * cap, 1, 128).reshape(B, Hkv, cap, 128)
        sv = synth.gen_values(rng, B * Hkv * cap, 1, 128).reshape(B, Hkv, cap, 128)
        sl = rng.integers(0, cap + 1, B).astype(np.int32)
        o.attend_mixed(T(q, torch.bfloat16), T(pt), T(np.asarray(L, np.int32)), T(pool), T(RK), T(RV),
                       T(sk, torch.bfloat16), T(sv, torch.bfloat16), T(sl), ws, out)
        ref, _ = O.attend_mixed(q, pt, L, pool, sk, sv, sl, RK, RV, fmt, Hkv)
    torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy() - ref).max() <= 2e-3


def test_attend_page_indirection_invariance():
    """Shuffling the physical pages (same logical cache) must not change the output."""
    torch = _torch()
    rng = np.random.default_rng(5)
    fmt = O.PageFormat(128, 2, 64, 64)
    pt, pool, RK, RV = _oracle_pool(rng, fmt, 2, 8, [700, 450], shuffle=False)
    q = synth.gen_decode_q(rng, 2, 32, 128)
    o = make()
    a, _, _ = _run_attend(o, q, pt, [700, 450], pool, RK, RV)
    perm = rng.permutation(pool.shape[0])
    pool2 = np.empty_like(pool)
    pool2[perm] = pool
    pt2 = perm[pt].astype(np.int32)
    b, _, _ = _run_attend(o, q, pt2, [700, 450], pool2, RK, RV)
    assert torch.equal(a, b)


def test_attend_full_size_sampled():
    """C2 at full size (B=16, L=32768, 32q/8kv, 2-bit, G=64) in the bench's launch
    configuration, on a synthetic random packed pool; two sequences checked against the
    oracle (all 32 heads each)."""
    torch = _torch()
    B, L, Hq, Hkv, P = 16, 32768, 32, 8, 64
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64)
    fmt = O.PageFormat(128, 2, 64, P)
    max_pages = L // P
    gen = torch.Generator(device="cuda").manual_seed(1)
    pool = synth.torch_random_pool(gen, B * max_pages, Hkv, o.page_bytes(), fmt.meta_off, P * 2, "cuda")
    rng = np.random.default_rng(1)
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    seq = np.full(B, L, np.int32)
    seq[5] = L - 1000
    ws = torch.empty(o.attend_workspace_bytes(B, max_pages), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    o.attend(T(q, torch.bfloat16), T(pt), T(seq), pool, T(RK), T(RV), ws, out)
    got = out.cpu().numpy()
    for b in [0, 5]:
        sub = pool[torch.from_numpy(pt[b].astype(np.int64)).cuda()].cpu().numpy()
        ref, _ = O.attend(q[b:b + 1], np.arange(max_pages, dtype=np.int32)[None], [seq[b]], sub, RK, RV,
                          fmt, Hkv)
        assert np.abs(got[b] - ref[0]).max() <= 2e-3


def test_attend_c4_full_size_sampled():
    """C4 at full size (g = 8: 64 q / 8 kv heads, 2-bit, G = 64, B = 16, L = 131072) in the
    bench's launch configuration on a random packed pool; one sequence (all 64 heads) against
    the oracle."""
    torch = _torch()
    B, L, Hq, Hkv, P = 16, 131072, 64, 8, 64
    o = make(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64)
    fmt = O.PageFormat(128, 2, 64, P)
    max_pages = L // P
    gen = torch.Generator(device="cuda").manual_seed(2)
    pool = synth.torch_random_pool(gen, B * max_pages, Hkv, o.page_bytes(), fmt.meta_off, P * 2, "cuda")
    rng = np.random.default_rng(2)
    pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    seq = np.full(B, L, np.int32)
    seq[3] = L - 5000
    ws = torch.empty(o.attend_workspace_bytes(B, max_pages), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
    o.attend(T(q, torch.bfloat16), T(pt), T(seq), pool, T(RK), T(RV), ws, out)
    got = out.cpu().numpy()
    b = 3
    sub = pool[torch.from_numpy(pt[b].astype(np.int64)).cuda()].cpu().numpy()
    ref, _ = O.attend(q[b:b + 1], np.arange(max_pages, dtype=np.int32)[None], [seq[b]], sub, RK, RV, fmt, Hkv)
    assert np.abs(got[b] - ref[0]).max() <= 2e-3


# ---------------------------------------------------------------------------- calibration
@pytest.mark.parametrize("variant,N,Hq,Hkv", [(0, 3000, 8, 2), (1, 3000, 8, 2), (0, 2500, 16, 2), (0, 9000, 2, 2)])
def test_calibration_parity_by_invariants(variant, N, Hq, Hkv):
    torch = _torch()
    rng = np.random.default_rng(21 + N + Hq)
    Q = synth.gen_queries(rng, N, Hq, Hkv, 128)
    SV = synth.gen_sv(rng, N, Hq, 128)
    o = make(num_q_heads=Hq, num_kv_heads=Hkv)
    o.set_variant(variant)
    acc = torch.zeros((Hkv, 2, 128, 128), dtype=torch.float64, device="cuda")
    o.calib_accumulate(T(Q[:1234], torch.bfloat16), T(SV[:1234], torch.bfloat16), acc)
    o.calib_accumulate(T(Q[1234:], torch.bfloat16), T(SV[1234:], torch.bfloat16), acc)
    ref = np.stack([O.cov_accumulate(Q, Hkv), O.cov_accumulate(SV, Hkv)], axis=1)
    got = acc.cpu().numpy()
    for h in range(Hkv):
        for w in range(2):
            assert np.linalg.norm(got[h, w] - ref[h, w]) / np.linalg.norm(ref[h, w]) <= 1e-5
    RK = torch.empty((Hkv, 128, 128), dtype=torch.float32, device="cuda")
    RV = torch.empty_like(RK)
    ev = torch.empty((Hkv, 2, 128), dtype=torch.float64, device="cuda")
    info = torch.empty((Hkv, 2), dtype=torch.int32, device="cuda")
    n_rows = N * (Hq // Hkv)
    o.calib_finalize(acc, Hkv, n_rows, RK, RV, ev, info)
    assert (info.cpu().numpy() > 0).all()
    H = O.hadamard(128)
    Pbr = H.T @ O.compose_rotation(np.eye(128))
    for h in range(Hkv):
        for w, R in enumerate([RK[h].cpu().numpy().astype(np.float64), RV[h].cpu().numpy().astype(np.float64)]):
            C = ref[h, w] / n_rows
            lam_o, U_o = O.eigh_desc(C)
            lam_g = ev[h, w].cpu().numpy()
            assert np.abs(R.T @ R - np.eye(128)).max() <= 1e-5                       # orthogonal
            d = np.diag(R.T @ C @ R)
            assert np.abs(d / (np.trace(C) / 128) - 1).max() <= 1e-5                  # Lemma
            U = R @ Pbr.T @ H.T                                                       # undo H P_br
            assert np.linalg.norm(C @ U - U * lam_g) / np.linalg.norm(C) <= 1e-5    # residual
            dC = np.linalg.norm(got[h, w] / n_rows - C, 2)
            assert np.abs(lam_g - lam_o).max() <= dC + 1e-6 * lam_o[0]                # Weyl
            gaps = np.minimum(np.abs(np.diff(lam_o, prepend=np.inf)), np.abs(np.diff(lam_o, append=-np.inf)))
            ok = gaps / lam_o[0] > 1e-3
            dots = np.abs(np.sum(U[:, ok] * U_o[:, ok], axis=0))
            assert (1 - dots).max() <= 1e-4                                           # Davis-Kahan
            assert np.all(np.diff(lam_g) <= 0)


def test_calibration_on_worked_example_spectrum():
    torch = _torch()
    rng = np.random.default_rng(4)
    lam = np.concatenate([[162.5, 85.5, 35.6, 17.4, 11.6, 7.5, 6.1, 5.0],
                          np.geomspace(4.9, 0.25, 112), [0.24, 0.22, 0.22, 0.20, 0.18, 0.05, 0.027, 0.009]])
    W = synth.haar(rng, 128)
    C = W @ np.diag(lam) @ W.T
    acc = torch.from_numpy(np.stack([C, C])[None]).cuda()
    o = make(num_q_heads=1, num_kv_heads=1)
    RK = torch.empty((1, 128, 128), dtype=torch.float32, device="cuda")
    RV = torch.empty_like(RK)
    ev = torch.empty((1, 2, 128), dtype=torch.float64, device="cuda")
    info = torch.empty((1, 2), dtype=torch.int32, device="cuda")
    o.calib_finalize(acc, 1, 1, RK, RV, ev, info)
    np.testing.assert_allclose(ev[0, 0].cpu().numpy(), np.sort(lam)[::-1], rtol=1e-9, atol=1e-12)
    R = RK[0].cpu().numpy().astype(np.float64)
    dg = np.diag(R.T @ C @ R)
    assert abs(dg.max() / dg.mean() - 1.0) < 1e-5                                     # 1.00
