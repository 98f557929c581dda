"""Per-call time of the decode path at the C2 shape, back to back over 8 layer pools (events only
at the two ends, so no per-call event commands): attend and decode_step at B = 16, attend at
B = 64 (per 16 sequences: the marginal streaming rate).  OSCAR_LIB selects the library build
(timing probes built with tools/build_variant.sh -DOSCAR_PROBE_...).  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17757_b200 import binding as Bnd, synth  # noqa: E402

HQ, HKV, D, P, NL = 32, 8, 128, 64, 8
BITS = int(os.environ.get("OSCAR_PROBE_BITS", "2"))
G = int(os.environ.get("OSCAR_PROBE_G", "64"))
dev = "cuda"
gen = torch.Generator(device=dev).manual_seed(3)
o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=BITS, group_size=G, page_size=P))
tok = 2 * (D * BITS // 8 + 4 * (D // G))
res = {"lib": os.environ.get("OSCAR_LIB", "default"), "bits": BITS, "G": G}
RK = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]
RV = [synth.torch_rotation(gen, HKV, D, dev) for _ in range(NL)]


def run(B, fn_name, L=32768, pps=0):
    mp = L // P
    oo = o if pps == 0 else Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=BITS, group_size=G,
                                                 page_size=P, attend_pages_per_split=pps))
    pools = [synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * 16 * BITS, P * (D // G), dev)
             for _ in range(NL)]
    pt = torch.randperm(B * mp, generator=gen, device=dev).to(torch.int32).reshape(B, mp).contiguous()
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    q = [synth.torch_decode_q(gen, B, HQ, D, dev) for _ in range(NL)]
    k = [synth.torch_keys(gen, B, HKV, D, dev) for _ in range(NL)]
    v = [synth.torch_values(gen, B, HKV, D, dev) for _ in range(NL)]
    ws = torch.empty(oo.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
    out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)

    def call(l):
        if fn_name == "attend":
            oo.attend(q[l], pt, sl, pools[l], RK[l], RV[l], ws, out)
        elif fn_name == "attend_norv":
            oo.attend(q[l], pt, sl, pools[l], RK[l], None, ws, out)
        else:
            oo.decode_step(q[l], k[l], v[l], pt, sl, pools[l], RK[l], RV[l], ws, out)
    for l in range(NL):
        call(l)
    torch.cuda.synchronize()
    if os.environ.get("OSCAR_PROBE_GRAPH"):
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(gr, stream=st):
                for _ in range(4):
                    for l in range(NL):
                        call(l)
        torch.cuda.current_stream().wait_stream(st)
        gr.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gr.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / (4 * NL))
        del pools
        return best, B * L * HKV * tok
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            for l in range(NL):
                call(l)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / (4 * NL))
    del pools
    torch.cuda.empty_cache()
    return best, B * L * HKV * tok


cases = os.environ.get("OSCAR_PROBE_CASES", "attend:16,attend_norv:16,decode_step:16,attend:64")
for case in cases.split(","):
    f = case.split(":")
    name, B = f[0], int(f[1])
    L = int(f[2]) if len(f) > 2 else 32768
    pps = int(f[3]) if len(f) > 3 else 0
    us, byt = run(B, name, L, pps)
    res[case + "_us"] = round(us, 2)
    res[case + "_TBps"] = round(byt / us / 1e6, 3)
print(json.dumps(res))
