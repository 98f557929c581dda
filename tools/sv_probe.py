"""Time oscar_calib_sv at the bench's calibration shape (8 sequences x 8192 tokens, 32 q / 8 kv heads,
causal) for both variants: python tools/sv_probe.py -> ms and TFLOP/s (causal flop count)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd  # noqa: E402

S, L, HQ, HKV, D = 8, 8192, 32, 8, 128
N = S * L
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(1)
Q = torch.randn((N, HQ, D), generator=g, device=dev).bfloat16()
K = torch.randn((N, HKV, D), generator=g, device=dev).bfloat16()
V = torch.randn((N, HKV, D), generator=g, device=dev).bfloat16()
starts = torch.arange(0, N, L, dtype=torch.int32, device=dev)
flops = 4.0 * D * HQ * S * L * (L + 1) / 2
outs = {}
for variant in (0, 1):
    o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV))
    o.set_variant(variant)
    SV = torch.empty((N, HQ, D), dtype=torch.bfloat16, device=dev)
    o.calib_sv(Q, K, V, starts, SV)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        o.calib_sv(Q, K, V, starts, SV)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    outs[variant] = SV.float()
    print(f"variant {variant}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
print("max |v0 - v1|", (outs[0] - outs[1]).abs().max().item())
