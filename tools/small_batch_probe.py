"""attend at small batch (C5 B in {1, 2, 4}), C2 shape, L = 32768: python tools/small_batch_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

L, HQ, HKV, D, P = 32768, 32, 8, 128, 64
G = int(os.environ.get("OSCAR_PROBE_G", "64"))   # group size (token-head bytes follow it)
PPS = int(os.environ.get("OSCAR_PROBE_PPS", "0"))  # attend_pages_per_split (0 = automatic)
dev = "cuda"
gen = torch.Generator(device=dev).manual_seed(3)
RK, RV = synth.torch_rotation(gen, HKV, D, dev), synth.torch_rotation(gen, HKV, D, dev)
for B in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "16"])]:
    o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=2, group_size=G, page_size=P,
                                 attend_pages_per_split=PPS))
    mp = L // P
    pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 32, P * (D // G), dev) for _ in range(4)]
    pt = torch.randperm(B * mp, generator=gen, device=dev).to(torch.int32).reshape(B, mp).contiguous()
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    q = synth.torch_decode_q(gen, B, HQ, D, dev)
    ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
    out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)
    for i in range(8):
        o.attend(q, pt, sl, pools[i % 4], RK, RV, ws, out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(12)]
    for i, (a, b) in enumerate(ev):
        a.record(); o.attend(q, pt, sl, pools[i % 4], RK, RV, ws, out); b.record()
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) for a, b in ev)[6] * 1e3
    byt = B * L * HKV * 2 * (32 + 4 * (D // G)) + 2 * B * HQ * D * 2
    print(f"B={B}: {us:.1f} us  {byt / us / 1e3:.0f} GB/s")
