"""Per-warp timeline of attend_partial_mma on the C2 workload (needs an OSCAR_TIMELINE build:
OSCAR_LIB=build_ab/liboscar_tl.so python tools/timeline_probe.py [decode])."""
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
NL = 4
pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 32, P * 2, dev) for _ in range(NL)]
pt = torch.arange(B * mp, dtype=torch.int32, device=dev).reshape(B, mp)
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
RK = synth.torch_rotation(gen, HKV, D, dev)
RV = synth.torch_rotation(gen, HKV, D, dev)
q = synth.torch_decode_q(gen, B, HQ, D, dev)
k = synth.torch_keys(gen, B, HKV, D, dev)
v = synth.torch_values(gen, B, HKV, D, dev)
ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)
dec = len(sys.argv) > 1 and sys.argv[1] == "decode"
for it in range(NL * 3):
    if dec:
        o.decode_step(q, k, v, pt, sl, pools[it % NL], RK, RV, ws, out)
    else:
        o.attend(q, pt, sl, pools[it % NL], RK, RV, ws, out)
torch.cuda.synchronize()
buf = np.zeros((8192, 5), np.uint64)
lib = Bnd._lib
lib.oscar_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.oscar_debug_timeline(buf.ctypes.data, buf.nbytes) == 0
n = int((buf[:, 2] > 0).sum())
t = buf[:n].astype(np.int64)
t0 = t[:, 0].min()
start, wait, end, pages, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3], t[:, 4]
print(f"warps {n}  pages/warp min {pages.min()} max {pages.max()} mean {pages.mean():.2f}")
print("start  us: min %.2f p50 %.2f p90 %.2f max %.2f" % (start.min(), *np.percentile(start, [50, 90]), start.max()))
print("wait   us: min %.2f p50 %.2f p90 %.2f max %.2f" % (wait.min(), *np.percentile(wait, [50, 90]), wait.max()))
print("end    us: min %.2f p10 %.2f p50 %.2f p90 %.2f max %.2f" % (end.min(), *np.percentile(end, [10, 50, 90]), end.max()))
rate = pages / np.maximum(end - wait, 1e-3)
print("pages/us per warp: p10 %.3f p50 %.3f p90 %.3f" % tuple(np.percentile(rate, [10, 50, 90])))
smend = np.zeros(sm.max() + 1)
smp = np.zeros(sm.max() + 1)
for i in range(n):
    smend[sm[i]] = max(smend[sm[i]], end[i])
    smp[sm[i]] += pages[i]
print("per-SM pages min %d max %d; per-SM last end min %.2f max %.2f" % (smp.min(), smp.max(), smend.min(), smend.max()))
hist, edges = np.histogram(end, bins=12)
print("end histogram:", " ".join(f"{e:.0f}:{h}" for e, h in zip(edges, hist)))
used = np.unique(sm)
first = np.array([end[sm == s].min() for s in used])
last = np.array([end[sm == s].max() for s in used])
pg = np.array([pages[sm == s].sum() for s in used])
nw = np.array([(sm == s).sum() for s in used])
rate_sm = pg / (last - wait.min())
print("SMs used %d; warps/SM %s" % (len(used), np.bincount(nw)))
print("per-SM pages/us: p10 %.2f p50 %.2f p90 %.2f min %.2f max %.2f" % (*np.percentile(rate_sm, [10, 50, 90]), rate_sm.min(), rate_sm.max()))
print("per-SM (last-first) end spread us: p50 %.2f p90 %.2f max %.2f" % (*np.percentile(last - first, [50, 90]), (last - first).max()))
for w in sorted(set(nw)):
    sel = nw == w
    print(f"  SMs with {w} warps: n={sel.sum()} pages/us mean {rate_sm[sel].mean():.2f}  last end mean {last[sel].mean():.1f}")
