"""Timeline of one decode step (C2 shape) from %globaltimer marks written by a probe build
(tools/build_variant.sh tl -DOSCAR_PROBE_TL; OSCAR_LIB=build_ab/liboscar_tl.so).  Layers run back
to back over 8 pools; the marks of one call in the middle (after warm-up) are printed relative to
the earliest prologue entry: per kernel kind, the quantiles of entry / after-wait / end times."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

HQ, HKV, D, P, NL, L = 32, 8, 128, 64, 8, 32768
B = int(os.environ.get("OSCAR_TL_B", "16"))
FN = os.environ.get("OSCAR_TL_FN", "decode_step")
dev = "cuda"
gen = torch.Generator(device=dev).manual_seed(3)
o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=2, group_size=64, page_size=P))
mp = L // P
RK = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
RV = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 32, P * 2, dev) for _ in range(NL)]
pt = torch.randperm(B * mp, generator=gen, device=dev).to(torch.int32).reshape(B, mp).contiguous()
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
q = [synth.torch_decode_q(gen, B, HQ, D, dev) for _ in range(NL)]
k = [synth.torch_keys(gen, B, HKV, D, dev) for _ in range(NL)]
v = [synth.torch_values(gen, B, HKV, D, dev) for _ in range(NL)]
ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)
tl = torch.zeros(3 * 32768, dtype=torch.int64, device=dev)
lib = Bnd._lib
lib.oscar_probe_timeline.argtypes = [ctypes.c_void_p]


def call(l):
    if FN == "attend":
        o.attend(q[l], pt, sl, pools[l], RK[l], RV[l], ws, out)
    else:
        o.decode_step(q[l], k[l], v[l], pt, sl, pools[l], RK[l], RV[l], ws, out)


for _ in range(3):
    for l in range(NL):
        call(l)
torch.cuda.synchronize()
for l in range(NL):
    if l == 4:
        lib.oscar_probe_timeline(ctypes.c_void_p(tl.data_ptr()))
    call(l)
    if l == 4:
        lib.oscar_probe_timeline(ctypes.c_void_p(0))
torch.cuda.synchronize()
t = tl.cpu().numpy().reshape(3, 8192, 4).astype(np.float64)
marks = t[t > 0]
t0 = marks.min()                              # earliest mark of any kernel (fused prologue: no kind-0 entry)
res = {"fn": FN}
for kind, name, slots in ((0, "prologue", ("entry", "after_wait", "end", "rotated")), (1, "partial", ("entry", "after_wait", "end")),
                          (2, "merge", ("entry", "pre_wait_done", "after_wait", "end"))):
    rows = t[kind][t[kind].max(axis=1) > 0]
    d = {"n": int(rows.shape[0])}
    for i, s in enumerate(slots):
        x = (rows[rows[:, i] > 0, i] - t0) / 1e3
        if x.size:
            d[s] = [round(float(np.quantile(x, qq)), 2) for qq in (0.0, 0.1, 0.5, 0.9, 1.0)]
    res[name] = d
print(json.dumps(res))
np.save(os.path.join("gpurun_out", f"timeline_{FN}_{os.path.basename(os.environ.get('OSCAR_LIB', 'default'))}.npy"), t)
