"""Pins of the CPU oracle against what the paper and the mathematics fix (not against itself).

Each test names the passage it follows.  Printed values come from tests/golden/ (copied from
PAPER.md, cited there).  CPU only.
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2605_17757_b200 import synth
from conftest import GOLDEN, load_worked_example


def scalars():
    out = {}
    with open(os.path.join(GOLDEN, "paper_scalars.txt")) as f:
        for ln in f:
            ln = ln.split("#")[0].strip()
            if ln:
                name, *vals = ln.split()
                out[name] = [float(v) for v in vals]
    return out


PS = scalars()
WE = {k: np.array(v) for k, v in load_worked_example().items()}


# ------------------------------------------------------------------ App A.1 Hadamard
def test_hadamard_closed_forms():
    assert np.array_equal(O.hadamard(1), np.ones((1, 1)))                      # H_1 = [1]
    s = 1 / math.sqrt(2)
    np.testing.assert_allclose(O.hadamard(2), [[s, s], [s, -s]], atol=1e-15)   # recursion
    np.testing.assert_allclose(O.hadamard(4)[3], [0.5, -0.5, -0.5, 0.5], atol=1e-15)
    for d in [2, 4, 8, 16, 32, 64, 128, 256, 512]:
        H = O.hadamard(d)
        assert np.abs(H.T @ H - np.eye(d)).max() < 1e-9
        assert np.abs(np.abs(H) - 1 / math.sqrt(d)).max() < 1e-12
    for bad in [0, 3, 6, 100]:
        with pytest.raises(ValueError):
            O.hadamard(bad)


def test_hadamard_order_pinned_by_printed_rows():
    """P:L163-171 -> P:L255-263 (raw · H = pure-Hadamard row) and P:L186-194 -> P:L209-217
    (K U_Q · H).  2-decimal printing bounds the error (max seen 0.011)."""
    H = O.hadamard(128)
    assert np.abs(WE["raw_K_t"] @ H - WE["K_H"]).max() < 0.02
    assert np.abs(WE["K_UQ"] @ H - WE["K_UQ_H"]).max() < 0.02
    # a column-sequency-ordered Walsh matrix would miss by O(1)-O(10)
    seq = np.argsort([np.sum(np.abs(np.diff(np.sign(H[:, j])))) for j in range(128)], kind="stable")
    assert np.abs(WE["raw_K_t"] @ H[:, seq] - WE["K_H"]).max() > 1.0


# ------------------------------------------------------------------ bit reversal / P_br
def test_bit_reversal_closed_form_and_printed_placement():
    assert list(O.bit_reversal(2)) == [0, 1]
    assert list(O.bit_reversal(8)) == [0, 4, 2, 6, 1, 5, 3, 7]
    assert list(O.pbr_placement(128)[:8]) == [int(v) for v in PS["placement_top1to8"]]
    for d in [2, 4, 8, 16, 32, 64, 128]:
        b = O.bit_reversal(d)
        assert np.array_equal(b[b], np.arange(d))                              # involution


def test_pbr_balance_every_power_of_two_group():
    """for any power-of-two G | d the top-d/G ranks land one per group."""
    for d in [2, 4, 8, 16, 32, 64, 128]:
        place = O.pbr_placement(d)
        G = 1
        while G <= d:
            groups = place[: d // G] // G
            assert len(set(groups.tolist())) == d // G
            G *= 2


def test_compose_pbr_convention_pinned_exactly():
    """P:L209-217 -> P:L232-240: step 3 is step 2 with out[j] = in[beta(j)], zero error
    ("the set of 128 values is identical")."""
    R0 = O.compose_rotation(np.eye(128))                  # = H_Had · P_br
    Pbr = O.hadamard(128).T @ R0
    assert np.abs(WE["K_UQ_H"] @ Pbr - WE["K_UQ_H_P"]).max() < 1e-12
    assert np.abs(WE["K_UQ"] @ R0 - WE["K_UQ_H_P"]).max() < 0.02
    assert sorted(WE["K_UQ_H"].tolist()) == sorted(WE["K_UQ_H_P"].tolist())


def test_rotate_pinned_by_printed_rows():
    """App A.5 P:L1229-1233 x̃ = x·R, row-vector convention, checked through O.rotate
    itself on the printed worked example: raw K_t · H = the printed pure-Hadamard row
    (P:L163 -> P:L255); K U_Q · H = P:L209-217; K U_Q · (H P_br) = the printed OSCAR row
    (P:L186 -> P:L232).  Two heads with different R pin the per-head indexing; the transposed
    operand (x · Rᵀ, what a swapped einsum would compute) is excluded by a cyclic-shift R."""
    H = O.hadamard(128)
    R0 = O.compose_rotation(np.eye(128))
    X = np.stack([WE["raw_K_t"], WE["K_UQ"], WE["K_UQ"]])[None]          # [T=1, heads=3, d]
    R = np.stack([H, H, R0]).astype(np.float32)
    out = O.rotate(X, R)
    assert out.dtype == np.float32 and out.shape == (1, 3, 128)
    assert np.abs(out[0, 0] - WE["K_H"]).max() < 0.02
    assert np.abs(out[0, 1] - WE["K_UQ_H"]).max() < 0.02
    assert np.abs(out[0, 2] - WE["K_UQ_H_P"]).max() < 0.02
    # H P_br is symmetric (P_br H P_br = H for Sylvester H), so the orientation x·R vs x·Rᵀ is
    # pinned by a non-symmetric closed form: R[k][(k+1) mod d] = 1 gives (x R)_j = x_{j-1}
    Sh = np.roll(np.eye(128, dtype=np.float32), 1, axis=1)
    sh = O.rotate(X[:, :1], Sh[None])
    assert np.array_equal(sh[0, 0], np.roll(WE["raw_K_t"], 1).astype(np.float32))
    # rows are independent (token axis): a second token equal to the first gives the same row
    out2 = O.rotate(np.concatenate([X, X * 2]), R)
    assert np.array_equal(out2[0], out[0]) and np.allclose(out2[1], 2 * out[0], rtol=1e-6, atol=1e-6)


def _beta(j, m):
    return int(format(j, f"0{m}b")[::-1], 2)


def test_calibrate_from_sums_closed_forms():
    """Alg. 1 Calibrate: C = acc / n_rows, EigVec descending, R = U H P_br
    (Eq. 3), R_K from the C_Q sums and R_V from the C_S sums.  Diagonal sums have
    U = a permutation known in closed form, so R and λ are written out independently with
    scipy's Sylvester Hadamard and a string bit reversal."""
    from scipy.linalg import hadamard as sylvester
    d, n = 128, 37
    Hs = sylvester(d) / math.sqrt(d)
    lam = np.linspace(9.0, 0.5, d)                     # distinct, descending
    acc_q = np.diag(lam * n)[None]                     # C_Q = diag(λ): U = I
    acc_s = np.diag(lam[::-1] * n)[None]               # C_S = diag(λ ascending): U = J (reversal)
    R_K, R_V, lam_q, lam_s = O.calibrate_from_sums(acc_q, acc_s, n)
    Rk_exp = np.empty((d, d))
    Rv_exp = np.empty((d, d))
    for j in range(d):
        Rk_exp[:, j] = Hs[:, _beta(j, 7)]              # (x U H P_br)_j = (x U H)_{β(j)}
        Rv_exp[:, j] = Hs[::-1, _beta(j, 7)]           # U = J reverses the rows of H
    assert np.abs(R_K[0] - Rk_exp).max() < 1e-7 and np.abs(R_V[0] - Rv_exp).max() < 1e-7
    np.testing.assert_allclose(lam_q[0], lam, rtol=1e-12)          # λ of acc / n_rows, descending
    np.testing.assert_allclose(lam_s[0], lam, rtol=1e-12)
    # a 4 x 4 case with a non-trivial eigenvector pair: [[3,1],[1,3]] ⊕ diag(1, 0.5)
    C4 = np.array([[3, 1, 0, 0], [1, 3, 0, 0], [0, 0, 1, 0], [0, 0, 0, 0.5]], float)
    R4, _, l4, _ = O.calibrate_from_sums((C4 * 5)[None], np.eye(4)[None], 5)
    s = 1 / math.sqrt(2)
    U = np.array([[s, s, 0, 0], [s, -s, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]])   # sign rule: ties -> first +
    UH = U @ (sylvester(4) / 2)
    exp = np.stack([UH[:, _beta(j, 2)] for j in range(4)], axis=1)
    np.testing.assert_allclose(l4[0], [4, 2, 1, 0.5], rtol=1e-12)
    assert np.abs(R4[0] - exp).max() < 1e-7


def test_quantizer_codes_are_the_real_arithmetic_round():
    """Reading Z4 pinned to App A.5's real arithmetic: with the stored (s16, m16),
    Q+ = clip(round((x - m16)/s16), 0, q_max) in exact rational arithmetic (Python fractions).
    The oracle's two fp32 roundings (RN(x - m16), RN(1/s16)) may only move t by |t|·2^-22, so
    codes agree except within that distance of a .5 boundary — and such cases are rare."""
    from fractions import Fraction
    rng = np.random.default_rng(44)
    for bits, G in [(2, 64), (3, 32), (4, 128)]:
        qmax = 2 ** bits - 1
        X = (rng.standard_normal((40, 128)) * rng.uniform(0.01, 20, (40, 1))).astype(np.float32)
        codes, s16, m16 = O.quantize_rows(X, bits, G)
        n_near = 0
        for r in range(X.shape[0]):
            for c in range(128):
                gi = c // G
                s = Fraction(float(s16[r, gi]))
                if s == 0:
                    assert codes[r, c] == 0
                    continue
                t = (Fraction(float(X[r, c])) - Fraction(float(m16[r, gi]))) / s
                k = math.floor(t + Fraction(1, 2))
                if t + Fraction(1, 2) == k and k % 2 == 1:   # exact tie -> even
                    k -= 1
                exp = min(max(k, 0), qmax)
                if codes[r, c] != exp:
                    frac = t - math.floor(t)
                    assert abs(float(frac) - 0.5) <= abs(float(t)) * 2.0 ** -22 + 1e-12, (bits, G, r, c)
                    n_near += 1
        assert n_near <= 2


def test_group_range_statistic_printed():
    for row, key in [("raw_K_t", "group_range_raw"), ("K_UQ", "group_range_UQ"),
                     ("K_UQ_H", "group_range_UQH"), ("K_UQ_H_P", "group_range_UQHP"),
                     ("K_H", "group_range_H")]:
        np.testing.assert_allclose(O.group_ranges(WE[row], 64), PS[key], atol=0.011)


# ------------------------------------------------------------------ App A.2 PCA / eigen
def test_eigh_desc_invariants_and_sign_convention():
    rng = np.random.default_rng(1)
    for d in [2, 5, 16, 128]:
        X = rng.standard_normal((3 * d, d)) * (np.arange(1, d + 1) ** -0.7)
        A = X.T @ X
        lam, U = O.eigh_desc(A)
        assert np.all(np.diff(lam) <= 0)
        assert np.abs(U.T @ U - np.eye(d)).max() < 1e-9
        assert np.linalg.norm(U @ np.diag(lam) @ U.T - A) / np.linalg.norm(A) < 1e-7
        for j in range(d):
            i = np.argmax(np.abs(U[:, j]))
            assert U[i, j] > 0
    lam, U = O.eigh_desc(np.diag([2.0, 1.0]))
    np.testing.assert_allclose(lam, [2, 1])
    np.testing.assert_allclose(U, np.eye(2), atol=1e-15)
    lam, U = O.eigh_desc(np.diag([1.0, 2.0]))
    np.testing.assert_allclose(U, [[0, 1], [1, 0]], atol=1e-15)


def test_ky_fan_proposition():
    """Proposition: max over UᵀU=I_r of tr(UᵀAU) = Σ top-r λ, attained by V_r."""
    rng = np.random.default_rng(13)
    d = 6
    X = rng.standard_normal((10, d))
    A = X.T @ X
    lam, U = O.eigh_desc(A)
    for r in range(1, d + 1):
        best = lam[:r].sum()
        assert abs(np.trace(U[:, :r].T @ A @ U[:, :r]) - best) < 1e-9 * best
        for _ in range(300):
            Z, _ = np.linalg.qr(rng.standard_normal((d, r)))
            assert np.trace(Z.T @ A @ Z) <= best + 1e-9 * best


# ------------------------------------------------------------------ Lemma
def test_hadamard_diagonal_equalization_lemma():
    H = O.hadamard(2)
    np.testing.assert_allclose(H.T @ np.diag([3.0, 1.0]) @ H, [[2, 1], [1, 2]], atol=1e-15)
    rng = np.random.default_rng(2)
    for d in [4, 32, 128]:
        Lam = np.diag(rng.exponential(size=d) ** 3)
        D = np.diag(O.hadamard(d).T @ Lam @ O.hadamard(d))
        assert np.abs(D - np.trace(Lam) / d).max() < 1e-9 * np.trace(Lam) / d


def _worked_example_spectrum():
    """A 128-eigenvalue spectrum with the printed head/tail and trace 443."""
    top, bot = np.array(PS["spectrum_top8"]), np.array(PS["spectrum_bottom8"])
    mid = np.geomspace(4.9, 0.25, 112)
    mid *= (PS["trace_CQ"][0] - top.sum() - bot.sum()) / mid.sum()
    return np.concatenate([top, np.sort(mid)[::-1], bot])


def test_importance_ratio_one_for_UQH_and_OSCAR():
    """Table `tab:worked-example-layer10` importance column: 1.00 for U_Q H and OSCAR
    (Lemma), > 1 for pure Hadamard; tr/d = 443/128 = 3.46."""
    rng = np.random.default_rng(3)
    lam = _worked_example_spectrum()
    W = synth.haar(rng, 128)
    C = W @ np.diag(lam) @ W.T
    _, U = O.eigh_desc(C)
    R = O.compose_rotation(U)
    diag = np.diag(R.T @ C @ R)
    assert abs(diag.max() / diag.mean() - PS["importance_ratio_UQH"][0]) < 1e-6
    assert abs(diag.mean() - PS["lemma_tr_over_d"][0]) < 0.005
    RH = O.hadamard(128)
    dH = np.diag(RH.T @ C @ RH)
    assert dH.max() / dH.mean() > 1.05


# ------------------------------------------------------------------ Theorem 1
def test_theorem1_bruteforce():
    """Identity pairing (R = U_Q, λ desc vs μ asc) is minimal over all d! permutations and
    over random orthogonal Z (proof P:L1377-1528, rearrangement inequality)."""
    Lam, E = np.diag([3.0, 1.0]), np.diag([1.0, 2.0])
    assert np.trace(Lam @ E) == 5.0
    Pi = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.trace(Pi.T @ Lam @ Pi @ E) == 7.0
    rng = np.random.default_rng(11)
    for d in [3, 5, 6]:
        for _ in range(40):
            X = rng.standard_normal((2 * d, d))
            C = X.T @ X
            lam, U = O.eigh_desc(C)
            E = np.diag(np.sort(rng.exponential(size=d)))            # ascending μ
            base = np.trace(U.T @ C @ U @ E)
            for perm in itertools.permutations(range(d)):
                P = np.eye(d)[:, perm]
                assert np.trace(P.T @ U.T @ C @ U @ P @ E) >= base - 1e-9 * abs(base)
            for _ in range(50):
                Z = synth.haar(rng, d)
                assert np.trace(Z.T @ C @ Z @ E) >= base - 1e-9 * abs(base)


# ------------------------------------------------------------------ App A.5 quantizer
def test_quantizer_closed_forms():
    c, s, m = O.quantize_rows(np.array([[0.0, 1.0, 2.0, 3.0]], np.float32), 2, 4)
    assert c.tolist() == [[0, 1, 2, 3]] and float(s[0, 0]) == 1.0 and float(m[0, 0]) == 0.0
    assert np.array_equal(O.dequantize_rows(c, s, m, 4), [[0, 1, 2, 3]])
    c, s, m = O.quantize_rows(np.array([[-1.0, 0.0, 1.0, 2.0]], np.float32), 2, 4)
    assert c.tolist() == [[0, 1, 2, 3]]
    assert np.array_equal(O.dequantize_rows(c, s, m, 4), [[-1, 0, 1, 2]])
    c, s, m = O.quantize_rows(np.array([[5.0, 5.0, 5.0, 5.0]], np.float32), 2, 4)  # Z2
    assert c.tolist() == [[0, 0, 0, 0]] and np.array_equal(O.dequantize_rows(c, s, m, 4), [[5] * 4])
    c, s, m = O.quantize_rows(np.arange(16, dtype=np.float32)[None], 4, 16)
    assert c.tolist() == [list(range(16))]


def test_quantizer_error_bound_and_idempotence():
    """|x - Q(x)| <= s/2 for an unclipped group, with the fp16-metadata
    slack of reading Z5; quantize∘dequantize is idempotent."""
    rng = np.random.default_rng(5)
    for bits in [2, 3, 4]:
        for G in [32, 64, 128]:
            X = (rng.standard_normal((400, 128)) * rng.uniform(0.01, 20, (400, 1))).astype(np.float32)
            c, s16, m16 = O.quantize_rows(X, bits, G)
            assert c.max() <= 2 ** bits - 1
            Xh = O.dequantize_rows(c, s16, m16, G)
            s = np.repeat(s16.astype(np.float64), G, axis=-1)
            m = np.repeat(m16.astype(np.float64), G, axis=-1)
            ulp16 = np.abs(np.spacing(m.astype(np.float16)).astype(np.float64))
            bound = s / 2 + ulp16 / 2 + 4 * np.abs(np.spacing(X.astype(np.float32))).astype(np.float64)
            assert np.all(np.abs(X - Xh) <= bound)
            c2, _, _ = O.quantize_rows(Xh.astype(np.float32), bits, G)
            assert np.array_equal(c, c2)


def test_residual_monotone_in_bits():
    rng = np.random.default_rng(6)
    X = rng.standard_normal((200, 128)).astype(np.float32)
    tr = []
    for bits in [2, 3, 4]:
        c, s, m = O.quantize_rows(X, bits, 64)
        tr.append(np.trace(O.residual_cov(X, O.dequantize_rows(c, s, m, 64))))
    assert tr[0] > tr[1] > tr[2]


def test_pack_closed_forms_and_roundtrip():
    assert O.pack_codes(np.array([0, 1, 2, 3], np.uint8), 2).tolist() == [0xE4]
    assert O.pack_codes(np.array([1, 2], np.uint8), 4).tolist() == [0x21]
    # 3-bit (reading Z36, worked by hand): low plane = the 2-bit stream of code & 3, high plane
    # bit of channel 16j + 4i + f at byte d/4 + 4(j // 2) + i, bit 4(j % 2) + f.  Codes 0..7 four
    # times: every low byte (0, 1, 2, 3) = 0xE4; the high bit is set exactly for i odd -> bytes
    # 0x00, 0xFF, 0x00, 0xFF.  A single code 4 on channel 5 (j 0, i 1, f 1) -> byte 9, bit 1.
    assert O.pack_codes(np.array(list(range(8)) * 4, np.uint8), 3).tolist() == [0xE4] * 8 + [0x00, 0xFF, 0x00, 0xFF]
    one = np.zeros(32, np.uint8)
    one[5] = 4
    assert O.pack_codes(one, 3).tolist() == [0] * 9 + [0x02, 0, 0]
    with pytest.raises(ValueError):
        O.pack_codes(np.zeros(8, np.uint8), 3)
    rng = np.random.default_rng(7)
    for bits in [2, 3, 4]:
        c = rng.integers(0, 2 ** bits, size=(20000, 128), dtype=np.uint8)
        assert np.array_equal(O.unpack_codes(O.pack_codes(c, bits), bits, 128), c)


def test_clip_closed_forms():
    x = np.array([[1.0, -2.0, 3.0, -4.0]], np.float32)
    assert np.array_equal(O.clip_rows(x, 1.0), x)                         # rho = 1 no-op
    assert O.clip_index(0.5, 4) == 1
    np.testing.assert_array_equal(O.clip_rows(x, 0.5), [[1, -2, 2, -2]])    # tau = 2
    z = np.zeros((1, 8), np.float32)
    assert np.array_equal(O.clip_rows(z, 0.9), z)
    assert O.clip_index(0.96, 128) == 122 and O.clip_index(0.92, 128) == 117


def test_worked_example_residual_soft_pin():
    """Table P:L282-286 tr(E_K) column (per-token means over 8000 tokens, reading Z28) vs the
    INT2 G=64 residual of the single printed token in each basis: same ordering of the
    extremes (U_Q worst, OSCAR best) and within 20%.  Soft pin."""
    res = []
    for row in ["raw_K_t", "K_H", "K_UQ", "K_UQ_H", "K_UQ_H_P"]:
        x = WE[row].astype(np.float32)[None]
        c, s, m = O.quantize_rows(x, 2, 64)
        res.append(float(np.sum((O.dequantize_rows(c, s, m, 64) - x) ** 2)))
    table = PS["table_trEK"]
    assert int(np.argmax(res)) == 2 and int(np.argmin(res)) == 4
    for r, t in zip(res, table):
        assert abs(r - t) / t < 0.2


# ------------------------------------------------------------------ BPE
def test_effective_bpe_printed():
    assert abs(O.effective_bpe(2, 128) - PS["bpe_naive_G128"][0]) < 1e-12
    assert abs(O.effective_bpe(2, 128, 320, 131072) - PS["bpe_oscar_128k"][0]) < 0.005
    assert abs(O.effective_bpe(2, 128, 320, 32768) - PS["bpe_oscar_32k"][0]) < 0.005
    assert abs(O.effective_bpe(4, 128) - PS["bpe_saw_int4"][0]) < 1e-12


# ------------------------------------------------------------------ Eq. (1), Eq. (2)
def test_eq1_logit_distortion_identity_through_oracle_quantizer():
    """‖QKᵀ − QK̂ᵀ‖²_F = tr(R_Kᵀ C_Q R_K E_K) with C_Q = QᵀQ unnormalized and E_K the residual
    covariance in the rotated frame, clipping included (Eq. 1)."""
    rng = np.random.default_rng(8)
    d, T, N = 64, 96, 80
    Q = synth.gen_queries(rng, N, 1, 1, d)[:, 0].astype(np.float64)
    K = synth.gen_keys(rng, T, 1, d)[:, 0].astype(np.float64)
    C = O.cov_accumulate(Q[:, None, :], 1)[0]
    _, U = O.eigh_desc(C / N)
    R = O.compose_rotation(U)                                   # fp64, orthogonal
    for rho in [1.0, 0.9]:
        Kr = K @ R
        Kc = O.clip_rows(Kr.astype(np.float32), rho)
        c, s, m = O.quantize_rows(Kc, 2, 32)
        Qd = O.dequantize_rows(c, s, m, 32)                     # Q(clip(x̃)) rotated frame
        Khat = Qd @ R.T
        lhs = np.linalg.norm(Q @ K.T - Q @ Khat.T) ** 2
        E = O.residual_cov(Kr, Qd)
        rhs = np.trace(R.T @ C @ R @ E)
        assert abs(lhs - rhs) / lhs < 1e-9


def test_eq2_and_cs_equals_VtStSV():
    """Eq. 2 and P:L1219: C_S from the rows of SV equals VᵀSᵀSV."""
    rng = np.random.default_rng(9)
    T, d = 24, 16
    Q = rng.standard_normal((T, 1, d))
    K = rng.standard_normal((T, 1, d))
    V = rng.standard_normal((T, 1, d))
    SV = O.score_value(Q, K, V, [T])[:, 0]
    logits = Q[:, 0] @ K[:, 0].T / math.sqrt(d)
    logits[np.triu(np.ones((T, T), bool), 1)] = -np.inf
    S = np.exp(logits - logits.max(1, keepdims=True))
    S /= S.sum(1, keepdims=True)
    np.testing.assert_allclose(SV, S @ V[:, 0], atol=1e-12)
    Cs = O.cov_accumulate(SV[:, None, :], 1)[0]
    np.testing.assert_allclose(Cs, V[:, 0].T @ S.T @ S @ V[:, 0], rtol=1e-10, atol=1e-12)
    Vh = V[:, 0] + 0.01 * rng.standard_normal((T, d))
    lhs = np.linalg.norm(S @ V[:, 0] - S @ Vh) ** 2
    rhs = np.trace((V[:, 0] - Vh).T @ S.T @ S @ (V[:, 0] - Vh))
    assert abs(lhs - rhs) / lhs < 1e-9


# ------------------------------------------------------------------ calibration targets
def test_covariance_targets_special_cases():
    rng = np.random.default_rng(10)
    Q = rng.standard_normal((50, 8, 16))                      # H_q = 8, H_kv = 2, g = 4
    acc = O.cov_accumulate(Q, 2)
    for h in range(2):
        assert abs(np.trace(acc[h]) - np.sum(Q[:, 4 * h:4 * h + 4] ** 2)) < 1e-9 * np.trace(acc[h])
    Z = np.zeros((5, 8, 16)); Z[:, 5, :] = 1.0                # q-head 5 belongs to kv head 1
    a = O.cov_accumulate(Z, 2)
    assert np.all(a[0] == 0) and np.all(a[1] == 5.0)
    Iso = np.eye(16)[None].repeat(1, 0).transpose(1, 0, 2) * 4.0   # 16 rows, 1 head
    np.testing.assert_allclose(O.cov_accumulate(Iso, 1)[0] / 16, np.eye(16))
    parts = [O.cov_accumulate(Q[i::3], 2) for i in range(3)]  # shard partials sum to whole
    np.testing.assert_allclose(sum(parts), acc, rtol=1e-12)
    same = np.repeat(Q[:, :1], 4, axis=1)                     # identical GQA heads
    np.testing.assert_allclose(O.cov_accumulate(same, 1)[0] / (50 * 4), O.cov_accumulate(Q[:, :1], 1)[0] / 50)


def test_score_value_special_cases():
    rng = np.random.default_rng(12)
    T, d = 7, 8
    V = rng.standard_normal((T, 1, d))
    K = rng.standard_normal((T, 1, d))
    SV = O.score_value(np.zeros((T, 1, d)), K, V, [T])         # equal logits: causal mean
    for i in range(T):
        np.testing.assert_allclose(SV[i, 0], V[: i + 1, 0].mean(0), atol=1e-12)
    SV1 = O.score_value(rng.standard_normal((1, 1, d)), K[:1], V[:1], [1])
    np.testing.assert_allclose(O.cov_accumulate(SV1, 1)[0], np.outer(V[0, 0], V[0, 0]))
    assert np.all(O.score_value(rng.standard_normal((T, 1, d)), K, 0 * V, [T]) == 0)
    two = O.score_value(np.zeros((6, 1, d)), K[:6], V[:6], [3, 3])   # block-diagonal
    np.testing.assert_allclose(two[3, 0], V[3, 0], atol=1e-12)


def test_calibration_scale_equivariance_and_orthogonality():
    rng = np.random.default_rng(14)
    Q = synth.gen_queries(rng, 300, 4, 2, 32)
    SV = synth.gen_sv(rng, 300, 4, 32)
    aq, as_ = O.cov_accumulate(Q, 2), O.cov_accumulate(SV, 2)
    RK, RV, lq, ls = O.calibrate_from_sums(aq, as_, 300 * 2)
    RK2, _, _, _ = O.calibrate_from_sums(aq * 9.0, as_, 300 * 2)
    np.testing.assert_allclose(RK, RK2, atol=1e-5)
    for R in list(RK) + list(RV):
        assert np.abs(R.astype(np.float64).T @ R - np.eye(32)).max() < 1e-6


# ------------------------------------------------------------------ attention
def test_attention_special_cases_and_bruteforce():
    rng = np.random.default_rng(15)
    d = 8
    RK, RV = synth.haar(rng, d), synth.haar(rng, d)
    v = rng.standard_normal((1, d))
    o, lse = O.attend_rows(rng.standard_normal(d), rng.standard_normal((1, d)), v, RK, RV, 0.3)
    np.testing.assert_allclose(o[0], v[0] @ RV.T, atol=1e-14)               # 1 token
    # softmax(0, ln 3) = (0.25, 0.75)
    Kr = np.zeros((2, d)); Kr[1, 0] = math.log(3.0)
    q = np.zeros(d); q[0] = 1.0
    Vr = rng.standard_normal((2, d))
    o, lse = O.attend_rows(q @ RK.T, Kr, Vr, RK, RV, 1.0)
    np.testing.assert_allclose(o[0], (0.25 * Vr[0] + 0.75 * Vr[1]) @ RV.T, atol=1e-14)
    assert abs(lse[0] - math.log(4.0)) < 1e-14
    # pass-through: rotated rows exact -> plain softmax attention, by direct loops
    for L in [1, 5, 16]:
        K = rng.standard_normal((L, d)); V = rng.standard_normal((L, d)); q = rng.standard_normal(d)
        o, lse = O.attend_rows(q, K @ RK, V @ RV, RK, RV, 1 / math.sqrt(d))
        w = [math.exp(sum(q[c] * K[t, c] for c in range(d)) / math.sqrt(d)) for t in range(L)]
        ref = [sum(w[t] * V[t, c] for t in range(L)) / sum(w) for c in range(d)]
        np.testing.assert_allclose(o[0], ref, atol=1e-12)
        assert abs(lse[0] - math.log(sum(w))) < 1e-12
        o1 = O.attend_alg1(q, K @ RK, V @ RV, RK, RV, 1 / math.sqrt(d))          # Alg. 1 form
        np.testing.assert_allclose(o1, o, atol=1e-12)
    o, lse = O.attend_rows(np.ones(d), np.zeros((0, d)), np.zeros((0, d)), RK, RV, 1.0)
    assert np.all(o == 0) and lse[0] == -np.inf


def test_page_format_and_paged_roundtrip():
    fmt = O.PageFormat(d=128, bits=2, G=64, P=64)
    assert fmt.page_bytes == 5120 and fmt.row_bytes == 32 and fmt.meta_off == 4096
    rng = np.random.default_rng(16)
    for bits, G in [(2, 64), (4, 32), (3, 128)]:
        fmt = O.PageFormat(d=128, bits=bits, G=G, P=64)
        H, T = 2, 150
        pool = np.zeros((8, H, fmt.page_bytes), np.uint8)
        Kr = rng.standard_normal((T, H, 128)).astype(np.float32)
        Vr = rng.standard_normal((T, H, 128)).astype(np.float32)
        slots = rng.permutation(8 * 64)[:T]
        O.quantize_rotated(Kr, Vr, slots, fmt, pool)
        for h in range(H):
            Kh, Vh = O.read_rows(pool, slots, h, fmt)
            c, s, m = O.quantize_rows(Kr[:, h], bits, G)
            np.testing.assert_array_equal(Kh, O.dequantize_rows(c, s, m, G))
            c, s, m = O.quantize_rows(Vr[:, h], bits, G)
            np.testing.assert_array_equal(Vh, O.dequantize_rows(c, s, m, G))
        # FORMAT placement: V bytes of a row are interleaved with stride 4 inside its 4-token
        # group, word order permuted; K rows of a 16-token tile are stored even-tokens-first
        page, off = divmod(int(slots[0]), 64)
        rb = fmt.row_bytes
        c, _, _ = O.quantize_rows(Vr[:1, 0], bits, G)
        packed = O.pack_codes(c, bits)[0]
        # word k of chunk (gid = j % 8): byte j of the 4 tokens of the row's group
        for j in ([0, 1, 7, 8, rb - 1] if bits != 3 else []):
            k = j // 8
            o = (fmt.vcodes_off + 16 * rb * (off // 16) + 16 * (32 * (k // 4) + 4 * (j % 8) + (off // 4) % 4)
                 + 4 * (k % 4) + off % 4)
            assert pool[page, 0, o] == packed[j]
        offs = np.concatenate([fmt.vbyte_offsets(u) for u in range(64)])
        assert len(set(offs.tolist())) == 64 * rb and offs.min() == fmt.vcodes_off \
            and offs.max() == fmt.vcodes_off + 64 * rb - 1                # a bijection on the region
        mo = [o for u in range(64) for g_ in range(128 // G) for o in fmt.meta_offsets(u, g_)]
        assert len(set(mo)) == len(mo) and min(mo) == fmt.meta_off
        assert max(mo) + 4 == fmt.meta_off + 64 * (128 // G) * 8 <= fmt.page_bytes
        c, _, _ = O.quantize_rows(Kr[:1, 0], bits, G)
        kpos = 16 * (off // 16) + 8 * (off % 2) + (off % 16) // 2
        assert np.array_equal(pool[page, 0, kpos * rb: (kpos + 1) * rb], O.pack_codes(c, bits)[0])


def test_paged_attend_matches_rows_and_alg1():
    rng = np.random.default_rng(17)
    fmt = O.PageFormat(d=128, bits=2, G=64, P=64)
    B, Hq, Hkv, L = 2, 4, 2, 100
    pt = synth.contiguous_page_table(B, 2, shuffle_rng=rng)
    pool = np.zeros((B * 2, Hkv, fmt.page_bytes), np.uint8)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    K, V = synth.gen_keys(rng, B * L, Hkv, 128), synth.gen_values(rng, B * L, Hkv, 128)
    pos = np.tile(np.arange(L), (B, 1))
    slots = synth.slots_for(pt, pos, 64).reshape(-1)
    O.quantize_append(K, V, slots, RK, RV, fmt, pool)
    q = synth.gen_decode_q(rng, B, Hq, 128)
    o, lse = O.attend(q, pt, [L, L - 37], pool, RK, RV, fmt, Hkv)
    Kh, Vh = O.read_rows(pool, slots[L:L + L - 37], 1, fmt)
    o1 = O.attend_alg1(q[1, 2:4], Kh, Vh, RK[1], RV[1], 1 / math.sqrt(128))
    np.testing.assert_allclose(o[1, 2:4], o1, atol=1e-12)


def test_attend_mixed_reduces_to_pure_cases():
    """NEXT-1 mixed cache (Alg. 1): with an empty bf16 segment it is
    `attend`; with an empty INT2 history it is plain softmax attention over the raw rows (direct
    loops)."""
    rng = np.random.default_rng(31)
    fmt = O.PageFormat(128, 2, 64, 64)
    B, Hq, Hkv, L, cap = 2, 4, 2, 150, 40
    pt = synth.contiguous_page_table(B, 3, shuffle_rng=rng)
    pool = np.zeros((B * 3, Hkv, fmt.page_bytes), np.uint8)
    RK, RV = synth.gen_rotation(rng, Hkv, 128), synth.gen_rotation(rng, Hkv, 128)
    for b in range(B):
        slots = synth.slots_for(pt[b:b + 1], np.arange(L)[None], 64).reshape(-1)
        O.quantize_append(synth.gen_keys(rng, L, Hkv, 128), synth.gen_values(rng, L, Hkv, 128),
                          slots, RK, RV, fmt, pool)
    q = synth.gen_decode_q(rng, B, Hq, 128, sigma=0.5)
    sk = synth.gen_keys(rng, B * Hkv * cap, 1, 128).reshape(B, Hkv, cap, 128)
    sv = synth.gen_values(rng, B * Hkv * cap, 1, 128).reshape(B, Hkv, cap, 128)
    o1, l1 = O.attend(q, pt, [L, 90], pool, RK, RV, fmt, Hkv)
    o2, l2 = O.attend_mixed(q, pt, [L, 90], pool, sk, sv, [0, 0], RK, RV, fmt, Hkv)
    np.testing.assert_allclose(o2, o1, atol=1e-12)
    np.testing.assert_allclose(l2, l1, atol=1e-12)
    o3, l3 = O.attend_mixed(q, pt, [0, 0], pool, sk, sv, [cap, 7], RK, RV, fmt, Hkv)
    d = 128
    for b, n in [(0, cap), (1, 7)]:
        for i in [0, 3]:
            h = i // 2
            w = [math.exp(sum(float(q[b, i, c]) * float(sk[b, h, t, c]) for c in range(d)) / math.sqrt(d))
                 for t in range(n)]
            ref = [sum(w[t] * float(sv[b, h, t, c]) for t in range(n)) / sum(w) for c in range(0, d, 17)]
            np.testing.assert_allclose(o3[b, i, ::17], ref, atol=1e-12)
            assert abs(l3[b, i] - math.log(sum(w))) < 1e-12


# ----------------------------------------------------------------------------------------
# CalibrateClip (Alg. 1, reading Z34)
def test_clip_surrogate_equals_explicit_logit_error():
    """The K surrogate tr(R^T C_Q R E_K) with C_Q = Q^T Q equals the squared logit error
    sum_{n,j} (q_n k_j^T - q_n khat_j^T)^2 computed from explicit queries (Eq. 1):
    khat_j = dequant(clip(k_j R)) R^T in the original frame."""
    rng = np.random.default_rng(5)
    d, N, Nq = 128, 96, 40
    Q = rng.standard_normal((Nq, d))
    K = (rng.standard_normal((N, d)) * np.where(np.arange(d) < 3, 9.0, 1.0)).astype(np.float32)
    R = np.linalg.qr(rng.standard_normal((d, d)))[0].astype(np.float32)
    grid = [0.9, 0.96, 1.0]
    obj = O.clip_objectives(K, R, Q.T @ Q, grid, 2, 64)
    Kr = O.rotate(K[:, None], R[None])[:, 0]
    for i, rho in enumerate(grid):
        c, s16, m16 = O.quantize_rows(O.clip_rows(Kr, rho), 2, 64)
        Khat = O.dequantize_rows(c, s16, m16, 64) @ R.astype(np.float64).T      # back to the K frame
        # logits against the rotated-then-unrotated exact keys (R orthogonal in fp64 up to fp32)
        Kexact = Kr.astype(np.float64) @ R.astype(np.float64).T
        err = Q @ (Kexact - Khat).T
        assert abs(obj[i] - (err ** 2).sum()) <= 1e-9 * (err ** 2).sum() + 1e-9


def test_calibrate_clip_provable_choices():
    """Channel 0 carries a planted outlier.  If the covariance target gives channel 0 no
    weight, clipping it costs nothing and shrinks every other channel's step, so rho < 1
    must win; if channel 0 dominates the weight, clipping error there dominates and rho = 1
    must win.  A singleton grid returns its value; equal-magnitude rows tie (first entry)."""
    rng = np.random.default_rng(6)
    d, N = 128, 64
    X = rng.standard_normal((N, 1, d)).astype(np.float32)
    X[:, 0, 0] = 100.0
    I = np.eye(d, dtype=np.float32)[None]
    w0 = np.eye(d)[None].copy(); w0[0, 0, 0] = 0.0              # channel 0 unweighted
    w1 = np.eye(d)[None].copy(); w1[0, 0, 0] = 1e6              # channel 0 dominant
    grid = [0.98, 1.0]
    _, rk, rv = O.calibrate_clip(X, X, I, I, w0, w1, grid, 2, 64)
    assert rk == 0.98 and rv == 1.0
    _, rk, rv = O.calibrate_clip(X, X, I, I, w0, w1, [1.0], 2, 64)
    assert rk == 1.0 and rv == 1.0
    Y = np.where(rng.random((N, 1, d)) < 0.5, -1.0, 1.0).astype(np.float32)    # |x| all equal
    obj, rk, rv = O.calibrate_clip(Y, Y, I, I, np.eye(d)[None], np.eye(d)[None], [0.9, 0.96], 2, 64)
    assert np.allclose(obj[..., 0], obj[..., 1]) and rk == 0.9 and rv == 0.9
