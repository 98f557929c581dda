"""GPU parity of the on-device S·V (Alg. 1, reading
Z16: causal incl. the diagonal, block-diagonal across sequences) against the fp64 oracle
`score_value`, and of C_S accumulated from it.  SV is stored in bf16 (the layout
oscar_calib_accumulate takes): elementwise bar = bf16 rounding (2^-8 relative) plus 2^-8 of the
largest |v| (the bf16 P operand: |Σ δp_t v_t| <= 2^-9 max|v|, with 2x margin)."""
import numpy as np
import pytest

import oracle as O
from paper_2605_17757_b200 import synth

pytestmark = pytest.mark.gpu


def T(x, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


@pytest.mark.parametrize("seq_lens,Hq,Hkv", [([300, 1, 77, 200], 8, 2), ([64], 4, 4), ([130, 260], 16, 2),
                                             ([1000, 129, 384], 8, 2)])
@pytest.mark.parametrize("variant", [0, 1])     # 0: tcgen05 kernel, 1: mma.sync kernel
def test_calib_sv_parity(seq_lens, Hq, Hkv, variant):
    import torch
    from paper_2605_17757_b200 import binding as B
    rng = np.random.default_rng(sum(seq_lens) + Hq)
    N = sum(seq_lens)
    Q = synth.gen_queries(rng, N, Hq, Hkv, 128)
    K = synth.gen_keys(rng, N, Hkv, 128)
    V = synth.gen_values(rng, N, Hkv, 128)
    ref = O.score_value(Q, K, V, seq_lens)
    starts = np.concatenate([[0], np.cumsum(seq_lens)[:-1]]).astype(np.int32)
    o = B.Oscar(B.Config(num_q_heads=Hq, num_kv_heads=Hkv))
    o.set_variant(variant)
    sv = torch.empty((N, Hq, 128), dtype=torch.bfloat16, device="cuda")
    o.calib_sv(T(Q, torch.bfloat16), T(K, torch.bfloat16), T(V, torch.bfloat16), T(starts), sv)
    got = sv.float().cpu().numpy()
    vmax = np.abs(V).max()
    err = np.abs(got - ref) - 2 ** -8 * np.abs(ref)
    assert err.max() <= 2 ** -8 * vmax, (err.max(), vmax)
    # C_S through oscar_calib_accumulate from the device SV vs the oracle's
    acc = torch.zeros((Hkv, 2, 128, 128), dtype=torch.float64, device="cuda")
    o.calib_accumulate(T(Q, torch.bfloat16), sv, acc)
    cs = acc[:, 1].cpu().numpy()
    cs_ref = O.cov_accumulate(ref, Hkv)
    assert np.linalg.norm(cs - cs_ref) <= 1e-2 * np.linalg.norm(cs_ref)


def test_shared_rotation_mode_accumulates_all_heads():
    """NEXT-4 shared rotations: a context with H_kv = 1 accumulates C_Q and C_S over
    all H_q query heads into one matrix (the oracle's cov_accumulate with one KV head), and
    finalize gives one orthogonal R shared by every head."""
    import torch
    from paper_2605_17757_b200 import binding as B
    rng = np.random.default_rng(3)
    N, Hq = 700, 32
    Q = synth.gen_queries(rng, N, Hq, 8, 128)
    SV = synth.gen_sv(rng, N, Hq, 128)
    o = B.Oscar(B.Config(num_q_heads=Hq, num_kv_heads=1))
    acc = torch.zeros((1, 2, 128, 128), dtype=torch.float64, device="cuda")
    o.calib_accumulate(T(Q, torch.bfloat16), T(SV, torch.bfloat16), acc)
    got = acc.cpu().numpy()
    for side, X in enumerate([Q, SV]):
        ref = O.cov_accumulate(X, 1)[0]
        assert np.linalg.norm(got[0, side] - ref) <= 1e-5 * np.linalg.norm(ref)
    RK = torch.empty((1, 128, 128), dtype=torch.float32, device="cuda")
    RV = torch.empty_like(RK)
    o.calib_finalize(acc, 1, N * Hq, RK, RV)
    R = RK[0].double().cpu().numpy()
    assert np.abs(R.T @ R - np.eye(128)).max() <= 1e-5
