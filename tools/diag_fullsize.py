"""Diagnostic: full-size C2 attend (random packed pool) vs the oracle on two sequences, for the
library selected by OSCAR_LIB, at several pages-per-split settings.  Prints max/mean abs error."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle as O
from paper_2605_17757_b200 import synth
from paper_2605_17757_b200 import binding as Bd

B, L, Hq, Hkv, P = 16, 32768, 32, 8, 64
fmt = O.PageFormat(128, 2, 64, P)
max_pages = L // P
gen = torch.Generator(device="cuda").manual_seed(1)
o0 = Bd.Oscar(Bd.Config(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64))
pool = synth.torch_random_pool(gen, B * max_pages, Hkv, o0.page_bytes(), fmt.meta_off, P * 2, "cuda")
rng = np.random.default_rng(1)
pt = synth.contiguous_page_table(B, max_pages, shuffle_rng=rng)
RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
q = synth.gen_decode_q(rng, B, Hq, 128)
seq = np.full(B, L, np.int32)
seq[5] = L - 1000
refs = {}
for b in [0, 5]:
    sub = pool[torch.from_numpy(pt[b].astype(np.int64)).cuda()].cpu().numpy()
    refs[b], _ = O.attend(q[b:b + 1], np.arange(max_pages, dtype=np.int32)[None], [seq[b]], sub, RK, RV, fmt, Hkv)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
for pps in [int(x) for x in os.environ.get('PPS', '0,4,9,16,32').split(',')]:
    for variant in [0, 1]:
        o = Bd.Oscar(Bd.Config(num_q_heads=Hq, num_kv_heads=Hkv, bits=2, group_size=64, attend_pages_per_split=pps))
        o.set_variant(variant)
        ws = torch.empty(o.attend_workspace_bytes(B, max_pages), dtype=torch.uint8, device="cuda")
        out = torch.empty((B, Hq, 128), dtype=torch.float32, device="cuda")
        o.attend(T(q).to(torch.bfloat16), T(pt), T(seq), pool, T(RK), T(RV), ws, out)
        got = out.cpu().numpy()
        errs = [np.abs(got[b] - refs[b][0]) for b in [0, 5]]
        worst = [np.unravel_index(e.argmax(), e.shape) for e in errs]
        print(f"lib={os.environ.get('OSCAR_LIB', 'default')} pps={pps} variant={variant} "
              f"max={max(e.max() for e in errs):.3e} mean={np.mean([e.mean() for e in errs]):.3e} "
              f"per-seq max={[f'{e.max():.2e}' for e in errs]} at(head,ch)={worst} "
              f"|o|={[f'{abs(refs[b][0][w]):.2f}' for b, w in zip([0, 5], worst)]}", flush=True)
