"""Debug helper: compare tensor-core vs CUDA-core covariance accumulation on the GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2605_17757_b200 import binding as B, synth
for (N, Hq, Hkv) in [(128, 1, 1), (256, 4, 1), (3000, 8, 2)]:
    rng = np.random.default_rng(1)
    Q = synth.gen_queries(rng, N, Hq, Hkv, 128)
    SV = synth.gen_sv(rng, N, Hq, 128)
    ref = np.stack([O.cov_accumulate(Q, Hkv), O.cov_accumulate(SV, Hkv)], axis=1)
    for v in [0, 1]:
        o = B.Oscar(B.Config(num_q_heads=Hq, num_kv_heads=Hkv)); o.set_variant(v)
        acc = torch.zeros((Hkv, 2, 128, 128), dtype=torch.float64, device="cuda")
        o.calib_accumulate(torch.from_numpy(Q).cuda().bfloat16(), torch.from_numpy(SV).cuda().bfloat16(), acc)
        got = acc.cpu().numpy()
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(N, Hq, Hkv, "variant", v, "rel", rel)
        if rel > 1e-4:
            d = got[0, 0] - ref[0, 0]
            i, j = np.unravel_index(np.argmax(np.abs(d)), d.shape)
            print("   max err at", i, j, got[0,0,i,j], ref[0,0,i,j], "diag ratio", np.diag(got[0,0])[:4] / np.diag(ref[0,0])[:4])
            print("   transposed?", np.linalg.norm(got[0,0].T - ref[0,0]) / np.linalg.norm(ref[0,0]))
