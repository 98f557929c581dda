"""Time the C2 prefill quantize_append (16 x 32768 tokens x 8 kv heads, 2-bit, G = 64) on the GPU
box: python tools/append_probe.py [G] [bits]  -> median ms and algorithmic GB/s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 64
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B, L, HKV, D, P = 16, 32768, 8, 128, 64
dev = "cuda"
o = Bnd.Oscar(Bnd.Config(num_q_heads=32, num_kv_heads=HKV, bits=bits, group_size=G, page_size=P))
gen = torch.Generator(device=dev).manual_seed(5)
T = B * L
K, V = synth.torch_keys(gen, T, HKV, D, dev), synth.torch_values(gen, T, HKV, D, dev)
npg = T // P
pool = torch.empty((npg, HKV, o.page_bytes()), dtype=torch.uint8, device=dev)
slots = (torch.randperm(npg, generator=gen, device=dev).repeat_interleave(P) * P + torch.arange(P, device=dev).repeat(npg))
RK, RV = synth.torch_rotation(gen, HKV, D, dev), synth.torch_rotation(gen, HKV, D, dev)
for _ in range(3):
    o.quantize_append(K, V, slots, RK, RV, pool)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(9)]
for a, b in ev:
    a.record(); o.quantize_append(K, V, slots, RK, RV, pool); b.record()
torch.cuda.synchronize()
ms = sorted(a.elapsed_time(b) for a, b in ev)[4]
byt = T * HKV * (2 * D * 2 + 2 * (D * bits // 8 + 4 * (D // G)) + 8 // HKV)
print(f"append G={G} b={bits}: {ms:.4f} ms  {byt / ms / 1e6:.0f} GB/s")
