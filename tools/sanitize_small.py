"""One small call of every kernel of liboscar.so, for compute-sanitizer:
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_small.py
Shapes are C1-like (oracle-sized) but take every kernel route: calibration (tcgen05 cov_accum,
Jacobi + compose, on-device S·V, CalibrateClip + selection), quantize_append (tcgen05 prefill
kernel, decode-size kernel, simple kernel with clipping), the stage hooks, attend (tensor-core
TQ and q-as-rows kernels, simple kernel, 3-bit), decode_step and attend_mixed, both variants.
Inputs are seeded and synthetic; results are not checked here (the parity tests do that)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

dev = "cuda"
gen = torch.Generator(device=dev).manual_seed(5)
D, P = 128, 64


def run(hq, hkv, bits, G, B, L, variant, clip=1.0):
    o = Bnd.Oscar(Bnd.Config(num_q_heads=hq, num_kv_heads=hkv, bits=bits, group_size=G, page_size=P,
                             clip_ratio_k=clip, clip_ratio_v=clip))
    o.set_variant(variant)
    # calibration
    N = 256
    Q = synth.torch_queries(gen, N, hq, hkv, D, dev)
    K = synth.torch_keys(gen, N, hkv, D, dev)
    V = synth.torch_values(gen, N, hkv, D, dev)
    SV = torch.empty((N, hq, D), dtype=torch.bfloat16, device=dev)
    o.calib_sv(Q, K, V, torch.tensor([0, 128], dtype=torch.int32, device=dev), SV)
    acc = torch.zeros((hkv, 2, D, D), dtype=torch.float64, device=dev)
    o.calib_accumulate(Q, SV, acc)
    RK = torch.empty((hkv, D, D), dtype=torch.float32, device=dev)
    RV = torch.empty_like(RK)
    info = torch.empty((hkv, 2), dtype=torch.int32, device=dev)
    o.calib_finalize(acc, hkv, N * (hq // hkv), RK, RV, None, info)
    o.calib_clip(K, V, RK, RV, acc, [0.9, 0.96, 1.0])
    # quantize_append: prefill (T = 300 crosses several 128-token tiles) and decode-size
    mp = (max(L) + P - 1) // P
    pool = torch.zeros((B * mp, hkv, o.page_bytes()), dtype=torch.uint8, device=dev)
    pt = torch.arange(B * mp, dtype=torch.int32, device=dev).reshape(B, mp).contiguous()
    for b in range(B):
        T = L[b]
        pos = torch.arange(T, device=dev)
        slots = (pt[b, pos // P].long() * P + pos % P).contiguous()
        if T:
            o.quantize_append(synth.torch_keys(gen, T, hkv, D, dev), synth.torch_values(gen, T, hkv, D, dev),
                              slots, RK, RV, pool)
    Xr = torch.empty((16, hkv, D), dtype=torch.float32, device=dev)
    o.rotate(synth.torch_keys(gen, 16, hkv, D, dev), RK, Xr)
    o.quantize_rotated(Xr, Xr, torch.arange(16, dtype=torch.int64, device=dev), pool)
    # attend, decode_step, attend_mixed
    seq = torch.tensor(L, dtype=torch.int32, device=dev)
    q = synth.torch_decode_q(gen, B, hq, D, dev)
    ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
    out = torch.empty((B, hq, D), dtype=torch.float32, device=dev)
    lse = torch.empty((B, hq), dtype=torch.float32, device=dev)
    o.attend(q, pt, seq, pool, RK, RV, ws, out, lse)
    o.decode_step(q, synth.torch_keys(gen, B, hkv, D, dev), synth.torch_values(gen, B, hkv, D, dev), pt, seq,
                  pool, RK, RV, ws, out)
    cap = 32
    sk = synth.torch_keys(gen, B * hkv * cap, 1, D, dev).reshape(B, hkv, cap, D)
    sv = synth.torch_values(gen, B * hkv * cap, 1, D, dev).reshape(B, hkv, cap, D)
    o.attend_mixed(q, pt, seq, pool, RK, RV, sk, sv, torch.full((B,), 20, dtype=torch.int32, device=dev), ws,
                   out, lse)
    torch.cuda.synchronize()


if os.environ.get("OSCAR_SANITIZE_ONE"):             # racecheck: one small case per kernel route
    run(8, 2, 2, 64, 2, [200, 33], 0)
    run(1, 1, 4, 32, 2, [130, 5], 0)
    run(8, 2, 3, 64, 1, [70], 1)
    print("sanitize_small: done")
    sys.exit(0)
for variant in (0, 1):
    run(32, 8, 2, 64, 3, [300, 77, 1], variant)            # C2-shaped heads: TQ kernel, tcgen05 append
    run(1, 1, 4, 32, 4, [256, 130, 64, 5], variant)         # C1 shape: q-as-rows kernel
    run(16, 2, 2, 64, 2, [200, 64], variant)                # g = 8 (two 8-combo tiles)
    run(8, 2, 3, 64, 2, [150, 20], variant)                 # 3-bit: simple kernels
run(8, 2, 2, 64, 2, [100, 33], 0, clip=0.96)                # clipping: simple append kernel
print("sanitize_small: done")
