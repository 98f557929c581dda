"""Check that the e2e leg's H2D/D2H copies are inside the timed region (C2, 32 layers)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

B, L, HQ, HKV, D, P, NL = 16, 32768, 32, 8, 128, 64, 8
dev = "cuda"
o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=2, group_size=64, page_size=P))
gen = torch.Generator(device=dev).manual_seed(3)
mp = L // P
pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 32, P * 2, dev) for _ in range(NL)]
pt = torch.arange(B * mp, dtype=torch.int32, device=dev).reshape(B, mp)
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
RK = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
RV = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
qs = [synth.torch_decode_q(gen, B, HQ, D, dev) for _ in range(NL)]
ks = [synth.torch_keys(gen, B, HKV, D, dev) for _ in range(NL)]
vs = [synth.torch_values(gen, B, HKV, D, dev) for _ in range(NL)]
ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
n_q, n_k = qs[0].numel(), ks[0].numel()
per = n_q + 2 * n_k
h_in = torch.cat([torch.cat([qs[l].reshape(-1), ks[l].reshape(-1), vs[l].reshape(-1)]) for l in range(NL)]).cpu().pin_memory()
d_in = torch.empty_like(h_in, device=dev)
d_out = torch.empty((NL, B, HQ, D), dtype=torch.bfloat16, device=dev)
h_out = torch.empty((NL, B, HQ, D), dtype=torch.bfloat16).pin_memory()
views = [(d_in[l * per:l * per + n_q].view(qs[l].shape), d_in[l * per + n_q:l * per + n_q + n_k].view(ks[l].shape),
          d_in[l * per + n_q + n_k:(l + 1) * per].view(vs[l].shape)) for l in range(NL)]


def step(copies):
    if copies:
        d_in.copy_(h_in, non_blocking=True)
    for l in range(NL):
        q, k, v = views[l]
        o.decode_step(q, k, v, pt, sl, pools[l], RK[l], RV[l], ws, d_out[l])
    if copies:
        h_out.copy_(d_out, non_blocking=True)


for c in (False, True, False, True):
    for _ in range(2):
        step(c)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        step(c)
    b.record(); torch.cuda.synchronize()
    print("copies" if c else "device", "%.3f ms/step" % (a.elapsed_time(b) / 10), "H2D bytes", h_in.numel() * 2)
