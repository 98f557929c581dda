"""GPU parity of the pre-rotated-V mode ("R_V can be absorbed into
W_V / W_O"): R_V = NULL means V rows are stored without rotation and attend returns õ in V's
own frame.  The oracle runs the plain definition with R_V = I (identity rotation), which is the
same computation.  Bars as test_gpu_parity.py."""
import numpy as np
import pytest

import oracle as O
from paper_2605_17757_b200 import synth

pytestmark = pytest.mark.gpu


def T(x, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def make(**kw):
    from paper_2605_17757_b200 import binding as B
    return B.Oscar(B.Config(**kw))


@pytest.mark.parametrize("variant,Tn,bits,G", [(0, 1000, 2, 64), (0, 10, 2, 64), (1, 300, 4, 32), (0, 700, 3, 64)])
def test_prerotated_v_append_and_attend(variant, Tn, bits, G):
    import torch
    rng = np.random.default_rng(90 + Tn + bits)
    Hq, H, P = 8, 2, 64
    fmt = O.PageFormat(128, bits, G, P)
    npages = (Tn + P - 1) // P
    K = synth.gen_keys(rng, Tn, H, 128)
    V = synth.gen_values(rng, Tn, H, 128)
    RK = synth.gen_rotation(rng, H, 128)
    I = np.broadcast_to(np.eye(128, dtype=np.float32), (H, 128, 128)).copy()
    slots = np.arange(Tn, dtype=np.int64)                 # sequence 0 owns pages 0 .. npages-1
    ref_pool = np.zeros((npages, H, fmt.page_bytes), np.uint8)
    O.quantize_append(K, V, slots, RK, I, fmt, ref_pool)
    o = make(num_q_heads=Hq, num_kv_heads=H, bits=bits, group_size=G)
    o.set_variant(variant)
    pool = torch.zeros((npages, H, o.page_bytes()), dtype=torch.uint8, device="cuda")
    o.quantize_append(T(K, torch.bfloat16), T(V, torch.bfloat16), T(slots), T(RK), None, pool)
    got = pool.cpu().numpy()
    from oracle.boundary import check_pool_flips                # every difference: a boundary flip
    check_pool_flips(got, {"K": O.rotate(K, RK), "V": O.rotate(V, I)}, slots, fmt)
    # attend from the oracle pool (isolates the attend path) with R_V = NULL
    pt = np.arange(npages, dtype=np.int32)[None]
    q = synth.gen_decode_q(rng, 1, Hq, 128)
    ref, ref_lse = O.attend(q, pt, [Tn], ref_pool, RK, I, fmt, H)
    ws = torch.empty(o.attend_workspace_bytes(1, npages), dtype=torch.uint8, device="cuda")
    out = torch.empty((1, Hq, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((1, Hq), dtype=torch.float32, device="cuda")
    o.attend(T(q, torch.bfloat16), T(pt), T(np.array([Tn], np.int32)), T(ref_pool), T(RK), None, ws, out, lse)
    torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy() - ref).max() <= 2e-3
    assert (np.abs(lse.cpu().numpy() - ref_lse) <= 1e-3 + 1e-4 * np.abs(ref_lse)).all()
