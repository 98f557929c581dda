"""A/B of quantize_append builds (OSCAR_LIB) at the C2 prefill shape: median of 5 after 2 warm-ups."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402
T, HKV, D = 524288, 8, 128
gen = torch.Generator(device="cuda").manual_seed(9)
res = {"lib": os.environ.get("OSCAR_LIB", "default")}
for bits, G in [(2, 64), (3, 64), (4, 64), (2, 128), (2, 32)]:
    o = Bnd.Oscar(Bnd.Config(num_q_heads=32, num_kv_heads=HKV, bits=bits, group_size=G, page_size=64))
    K, V = synth.torch_keys(gen, T, HKV, D, "cuda"), synth.torch_values(gen, T, HKV, D, "cuda")
    R = synth.torch_rotation(gen, HKV, D, "cuda")
    pool = torch.empty((T // 64, HKV, o.page_bytes()), dtype=torch.uint8, device="cuda")
    slots = torch.arange(T, dtype=torch.int64, device="cuda")
    for _ in range(2):
        o.quantize_append(K, V, slots, R, R, pool)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a, b in ev:
        a.record(); o.quantize_append(K, V, slots, R, R, pool); b.record()
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) for a, b in ev)[2] * 1e3
    tok = 2 * (D * bits // 8 + 4 * (D // G))
    res[f"b{bits}G{G}_us"] = round(us, 1)
    res[f"b{bits}G{G}_frac"] = round(T * HKV * (512 + tok + 1) / us / 1e3 / 6536.4, 3)
    del K, V, pool
print(json.dumps(res))
