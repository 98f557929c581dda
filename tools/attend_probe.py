"""Time oscar_attend / oscar_decode_step variants on the C2 decode workload (GPU box):
python tools/attend_probe.py  ->  per-call µs for attend with R_V, attend with R_V = NULL
(no un-rotation: isolates the merge's R_V work) and decode_step.  OSCAR_PROBE_BITS picks the
code width (default 2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

B, L, HQ, HKV, D, P, NL = 16, 32768, 32, 8, 128, 64, 8
BITS = int(os.environ.get("OSCAR_PROBE_BITS", "2"))
dev = "cuda"
o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=BITS, group_size=64, page_size=P))
gen = torch.Generator(device=dev).manual_seed(3)
mp = L // P
pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 16 * BITS, P * 2, dev) for _ in range(NL)]
pt = torch.arange(B * mp, dtype=torch.int32, device=dev).reshape(B, mp)
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
RK = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
RV = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
q = [synth.torch_decode_q(gen, B, HQ, D, dev) for _ in range(NL)]
k = [synth.torch_keys(gen, B, HKV, D, dev) for _ in range(NL)]
v = [synth.torch_values(gen, B, HKV, D, dev) for _ in range(NL)]
ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)


def timeit(fn, reps=5):
    for l in range(NL):
        fn(l)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(NL * reps)]
    for r in range(reps):
        for l in range(NL):
            a, b = ev[r * NL + l]
            a.record()
            fn(l)
            b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return ts[len(ts) // 2]


print("attend      %.2f us" % timeit(lambda l: o.attend(q[l], pt, sl, pools[l], RK[l], RV[l], ws, out)))
print("attend R_V=0 %.2f us" % timeit(lambda l: o.attend(q[l], pt, sl, pools[l], RK[l], None, ws, out)))
print("decode_step %.2f us" % timeit(lambda l: o.decode_step(q[l], k[l], v[l], pt, sl, pools[l], RK[l], RV[l], ws, out)))

if len(sys.argv) > 1:      # pages-per-split sweep: python tools/attend_probe.py 8 16 32
    for pps in map(int, sys.argv[1:]):
        o2 = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=BITS, group_size=64, page_size=P,
                                  attend_pages_per_split=pps))
        ws2 = torch.empty(o2.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
        print("pps %2d attend %.2f us" % (pps, timeit(lambda l: o2.attend(q[l], pt, sl, pools[l], RK[l], RV[l], ws2, out))))
