"""The two rotation forms of the north star, stage for stage: oscar_rotate (dense
[x x]·[R_hi; R_lo] tcgen05 GEMM, fp32 rows out) vs oscar_rotate_fwht (the same GEMM with U, then the
Walsh–Hadamard transform + bit-reversed scatter in the epilogue), and the production
quantize_append for reference, at the C2 prefill shape (524288 tokens x 8 KV heads, K only for the
hooks).  Median of 5 CUDA-event timings after 2 warm-ups; one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

T, HKV, D = int(os.environ.get("OSCAR_ROT_T", 524288)), 8, 128
dev = "cuda"
gen = torch.Generator(device=dev).manual_seed(9)
o = Bnd.Oscar(Bnd.Config(num_q_heads=32, num_kv_heads=HKV, bits=2, group_size=64, page_size=64))
X = synth.torch_keys(gen, T, HKV, D, dev)
V = synth.torch_values(gen, T, HKV, D, dev)
R = synth.torch_rotation(gen, HKV, D, dev)
out = torch.empty((T, HKV, D), dtype=torch.float32, device=dev)
pool = torch.empty((T // 64, HKV, o.page_bytes()), dtype=torch.uint8, device=dev)
slots = torch.arange(T, dtype=torch.int64, device=dev)


def med(fn, reps=5):
    for _ in range(2):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2] * 1e3


res = {"T": T, "kv_heads": HKV}
res["rotate_dense_us"] = med(lambda: o.rotate(X, R, out))
res["rotate_fwht_us"] = med(lambda: o.rotate_fwht(X, R, out))
res["quantize_append_us"] = med(lambda: o.quantize_append(X, V, slots, R, R, pool))
hook_bytes = T * HKV * D * (2 + 4)          # bf16 in, fp32 out (K only)
res["rotate_dense_GBps"] = hook_bytes / res["rotate_dense_us"] / 1e3
res["rotate_fwht_GBps"] = hook_bytes / res["rotate_fwht_us"] / 1e3
print(json.dumps(res))
