"""Prologue phase timeline (needs an -DOSCAR_PTL build): OSCAR_LIB=build_ab/liboscar_ptl.so
python tools/merge_timeline.py  -> per-phase µs (median / max over CTAs) relative to the first
CTA start: launch, griddepcontrol.wait, split combine, smem combine, R_V wait, end."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

B, L, HQ, HKV, D, P = 16, 32768, 32, 8, 128, 64
dev = "cuda"
o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=2, group_size=64, page_size=P))
gen = torch.Generator(device=dev).manual_seed(3)
mp = L // P
pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 32, P * 2, dev) for _ in range(4)]
pt = torch.arange(B * mp, dtype=torch.int32, device=dev).reshape(B, mp)
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
RK, RV = synth.torch_rotation(gen, HKV, D, dev), synth.torch_rotation(gen, HKV, D, dev)
q = synth.torch_decode_q(gen, B, HQ, D, dev)
kn, vn = synth.torch_keys(gen, B, HKV, D, dev), synth.torch_values(gen, B, HKV, D, dev)
ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
for it in range(12):
    if it == 11:
        s0.record()
    o.decode_step(q, kn, vn, pt, sl, pools[it % 4], RK, RV, ws, out)
s1.record()
torch.cuda.synchronize()
print("last decode_step call %.2f us" % (s0.elapsed_time(s1) * 1e3))
buf = np.zeros((4096, 6), np.uint64)
lib = Bnd._lib
lib.oscar_debug_ptl.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.oscar_debug_ptl(buf.ctypes.data, buf.nbytes) == 0
t = buf[:B * HKV].astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "rows+R loaded", "partial dots", "16-way reduce", "quantize+append", "end (fragments)"]
for k, n in enumerate(names):
    x = (t[:, k] - t0) / 1e3
    print(f"{n:14s} min {x.min():7.2f}  p50 {np.median(x):7.2f}  max {x.max():7.2f} us")
