"""OSCAR oracle (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Each function transcribes one step of the paper, in the paper's order and notation,
fp64 unless the step fixes another precision (the fp32/fp16 quantizer steps of reading
Z4).  Library primitives used as single steps: ``np.linalg.eigh`` (the EigVec of
Alg. 1), matrix products, sorts.  No blocking, fusion or reordering.

Row-vector convention throughout: x̃ = x·R.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "hadamard", "bit_reversal", "eigh_desc", "compose_rotation", "pbr_placement",
    "cov_accumulate", "score_value", "calibrate_from_sums", "rotate", "clip_index",
    "clip_rows", "quantize_rows", "quantize_rows_detail", "dequantize_rows", "pack_codes", "unpack_codes",
    "PageFormat", "quantize_rotated", "quantize_append", "read_codes", "read_rows", "attend_rows",
    "attend", "attend_mixed", "attend_alg1", "residual_cov", "group_ranges", "effective_bpe",
    "clip_objectives", "calibrate_clip",
]


# ----------------------------------------------------------------------------------
# App A.1: normalized Walsh-Hadamard, Sylvester recursion
# H_1 = [1], H_2m = (1/sqrt 2) [[H_m, H_m], [H_m, -H_m]].  Natural (Sylvester) order is
# pinned by the worked example (raw row · H = printed pure-Hadamard row, P:L163 -> L255).
# ----------------------------------------------------------------------------------
def hadamard(d: int) -> np.ndarray:
    if d < 1 or d & (d - 1):
        raise ValueError(f"Hadamard dimension must be a power of two, got {d}")
    H = np.ones((1, 1), dtype=np.float64)
    while H.shape[0] < d:
        H = np.block([[H, H], [H, -H]]) / math.sqrt(2.0)
    return H


# Appendix `app:intuition_uhp`: beta = bit-reversal permutation on {0..d-1}.
def bit_reversal(d: int) -> np.ndarray:
    if d < 1 or d & (d - 1):
        raise ValueError(f"bit reversal needs a power of two, got {d}")
    m = d.bit_length() - 1
    out = np.zeros(d, dtype=np.int64)
    for k in range(d):
        r = 0
        for b in range(m):
            if k >> b & 1:
                r |= 1 << (m - 1 - b)
        out[k] = r
    return out


# "P_K places the eigenvector with the k-th largest eigenvalue at position
# beta(k)" -> placement list (top-1 -> 0, top-2 -> 64, ...).
def pbr_placement(d: int) -> np.ndarray:
    return bit_reversal(d)


# ----------------------------------------------------------------------------------
# App A.2 / Alg. 1: C = U Λ Uᵀ with λ_1 >= ... >= λ_d.
# Reading Z12: ties in λ keep ascending original index (stable sort);
# each eigenvector column is sign-flipped so its largest-|entry| is positive, ties to
# the lowest index.
# ----------------------------------------------------------------------------------
def eigh_desc(C: np.ndarray):
    C = np.asarray(C, dtype=np.float64)
    lam, U = np.linalg.eigh(C)              # LAPACK (ascending) — library step
    order = np.argsort(-lam, kind="stable")  # descending
    lam = lam[order]
    U = U[:, order].copy()
    for j in range(U.shape[1]):
        i = int(np.argmax(np.abs(U[:, j])))  # first index on ties
        if U[i, j] < 0:
            U[:, j] = -U[:, j]
    return lam, U


# ----------------------------------------------------------------------------------
# Eq. (3) / App intuition: R = U · H_Had · P_br.
# P_br is the pure bit-reversal of output columns: (x U H P_br)_j = (x U H)_{beta(j)}
# (reading Z10; pinned exactly by printed rows P:L209-217 -> P:L232-240).
# ----------------------------------------------------------------------------------
def compose_rotation(U: np.ndarray) -> np.ndarray:
    d = U.shape[0]
    H = hadamard(d)
    beta = bit_reversal(d)
    P = np.zeros((d, d), dtype=np.float64)
    for j in range(d):
        P[beta[j], j] = 1.0
    return np.asarray(U, dtype=np.float64) @ H @ P


# ----------------------------------------------------------------------------------
# §3 and the worked example's production metric:
# C_Q[h] ∝ Σ_n Σ_{i in G_h} q_{n,i}ᵀ q_{n,i}; query head i belongs to KV head i // g.
# The same accumulation on the rows of SV gives C_S (reading Z15).
# Returned UNNORMALIZED (reading Z13; Eq. 1 uses QᵀQ unnormalized, P:L9).
# ----------------------------------------------------------------------------------
def cov_accumulate(X: np.ndarray, num_kv_heads: int) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    N, Hq, d = X.shape
    if Hq % num_kv_heads:
        raise ValueError("H_q must be a multiple of H_kv")
    g = Hq // num_kv_heads
    acc = np.zeros((num_kv_heads, d, d), dtype=np.float64)
    for h in range(num_kv_heads):
        Xh = X[:, h * g:(h + 1) * g, :].reshape(N * g, d)
        acc[h] = Xh.T @ Xh
    return acc


# §3, Alg. 1: S = softmax_row(Q Kᵀ/√d + M); the C_S input is SV
# (VᵀSᵀSV = (SV)ᵀ(SV)).  M is causal including the diagonal and
# block-diagonal across calibration sequences (reading Z16).  Small cases only.
def score_value(Q: np.ndarray, K: np.ndarray, V: np.ndarray, seq_lens, scale=None) -> np.ndarray:
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    N, Hq, d = Q.shape
    Hkv = K.shape[1]
    g = Hq // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    SV = np.zeros((N, Hq, d), dtype=np.float64)
    start = 0
    for L in seq_lens:
        for i in range(Hq):
            h = i // g
            q = Q[start:start + L, i, :]
            k = K[start:start + L, h, :]
            v = V[start:start + L, h, :]
            logits = scale * (q @ k.T)
            mask = np.triu(np.ones((L, L), dtype=bool), k=1)
            logits[mask] = -np.inf
            logits -= logits.max(axis=1, keepdims=True)
            S = np.exp(logits)
            S /= S.sum(axis=1, keepdims=True)
            SV[start:start + L, i, :] = S @ v
        start += L
    return SV


# Alg. 1 `Calibrate` from accumulated sums: C = acc / n_rows, eigen-
# decompose (descending), compose R = U H P_br.  R is emitted as fp32 (RNE).
def calibrate_from_sums(acc_q: np.ndarray, acc_s: np.ndarray, n_rows: int):
    outs = []
    for acc in (acc_q, acc_s):
        Rs, lams = [], []
        for C in np.asarray(acc, dtype=np.float64):
            lam, U = eigh_desc(C / float(n_rows))
            Rs.append(compose_rotation(U))
            lams.append(lam)
        outs.append((np.array(Rs).astype(np.float32), np.array(lams)))
    (R_K, lam_q), (R_V, lam_s) = outs
    return R_K, R_V, lam_q, lam_s


# ----------------------------------------------------------------------------------
# App A.5 / Alg. 1: x̃ = x R.  Defined as the fp64 dot of the
# bf16 input with the fp32 R, rounded once to fp32 (RNE) — the "fp32 rotated values".
# X [T, H, d] (bf16-representable values), R [H, d, d].
# ----------------------------------------------------------------------------------
def rotate(X: np.ndarray, R: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    R = np.asarray(R, dtype=np.float32).astype(np.float64)
    return np.einsum("thd,hde->the", X, R).astype(np.float32)


# App A.5: tau_t = quantile_rho(|x̃_t,c|) over the whole row; reading Z6:
# nearest rank on the sorted |x̃|, index ceil(rho·d) - 1, rho taken as its fp32 value.
def clip_index(rho: float, d: int) -> int:
    return int(math.ceil(float(np.float32(rho)) * d)) - 1


def clip_rows(Xr: np.ndarray, rho: float) -> np.ndarray:
    Xr = np.asarray(Xr, dtype=np.float32)
    if float(np.float32(rho)) >= 1.0:
        return Xr.copy()
    d = Xr.shape[-1]
    k = clip_index(rho, d)
    tau = np.sort(np.abs(Xr), axis=-1)[..., k:k + 1]
    return np.minimum(np.maximum(Xr, -tau), tau).astype(np.float32)


# ----------------------------------------------------------------------------------
# App A.5: per-token, per-group asymmetric min-max quantizer,
# q_max = 2^b - 1, s = (max - min)/q_max, Q+ = clip(round(x/s + z), 0, q_max).
# Reading Z2/Z3/Z4: store (s16, m16) = fp16_rne(s), fp16_rne(min) (m = -s·z), and
# compute codes from the STORED metadata with this exact operation order:
#   s = (mx - mn) / q_max          [fp32 sub RN, fp32 div RN]
#   inv = 1 / float(s16)  (0 if s16 == 0)
#   dx = x - float(m16)             [fp32 sub RN]
#   c = clamp(rint_half_even(dx·inv exactly), 0, q_max)      (readings Z1, Z4)
# Returns codes uint8 [..., d], s16, m16 float16 [..., d/G].
# ----------------------------------------------------------------------------------
def quantize_rows(Xc: np.ndarray, bits: int, G: int):
    codes, s16, m16, _, _ = quantize_rows_detail(Xc, bits, G)
    return codes, s16, m16


def quantize_rows_detail(Xc: np.ndarray, bits: int, G: int):
    """quantize_rows plus its intermediates: the fp32 scale s before the fp16 store [..., d/G] and
    the exact pre-round value t = RN32(x - m16)·inv [..., d] (reading Z4), for checking that a
    differing GPU code or metadata value sits on a rounding boundary."""
    Xc = np.asarray(Xc, dtype=np.float32)
    d = Xc.shape[-1]
    if d % G:
        raise ValueError("G must divide d")
    qmax = np.float32(2 ** bits - 1)
    Xg = Xc.reshape(Xc.shape[:-1] + (d // G, G))
    mn = Xg.min(axis=-1)
    mx = Xg.max(axis=-1)
    s = (mx - mn) / qmax                      # fp32 RN, fp32 RN
    s16 = s.astype(np.float16)                # RNE
    m16 = mn.astype(np.float16)               # RNE
    s32 = s16.astype(np.float32)
    inv = np.where(s32 > 0, np.float32(1.0) / np.where(s32 > 0, s32, np.float32(1.0)), np.float32(0.0))
    inv = inv.astype(np.float32)
    dx = Xg - m16.astype(np.float32)[..., None]                      # fp32 RN
    # reading Z4: the product dx·inv is taken exactly (fp32 x fp32 fits fp64's 53 bits) and
    # rounded once, to the nearest integer (half-even) -- P:L1286-1295's real-arithmetic round
    t = dx.astype(np.float64) * inv.astype(np.float64)[..., None]
    c = np.clip(np.rint(t), 0, qmax).astype(np.uint8)               # np.rint = half-even
    return c.reshape(Xc.shape), s16, m16, s, t.reshape(Xc.shape)


# Q(x) = s (Q+ - z) = s16·c + m16, evaluated in fp64.
def dequantize_rows(codes: np.ndarray, s16: np.ndarray, m16: np.ndarray, G: int) -> np.ndarray:
    c = np.asarray(codes, dtype=np.float64)
    d = c.shape[-1]
    cg = c.reshape(c.shape[:-1] + (d // G, G))
    x = s16.astype(np.float64)[..., None] * cg + m16.astype(np.float64)[..., None]
    return x.reshape(c.shape)


# P:L560 "four 2-bit values packed per byte"; reading Z22: code i of a row occupies bits
# [b·i, b·i + b) of the row's little-endian bitstream (byte j = bits 8j..8j+7, LSB first), for
# b in {2, 4}.  Reading Z36 (b = 3, a byte-aligned layout so the decode kernel's integer tensor-
# core operands take the codes in place): the row is two planes — bytes [0, d/4) the 2-bit
# bitstream of the low bits (code & 3), bytes [d/4, d/4 + d/8) the high bits (code >> 2), the high
# bit of channel c = 16·j + 4·i + f (0 <= i, f < 4) at byte d/4 + 4·(j // 2) + i, bit 4·(j % 2) + f
# (d a multiple of 32).  Same bits per row; only their positions differ.
def _bit_position(i: int, k: int, bits: int, d: int):
    """(byte, bit) of bit k of code i inside a packed row."""
    if bits != 3:
        pos = bits * i + k
        return pos // 8, pos % 8
    if k < 2:                                   # low plane: the 2-bit bitstream
        pos = 2 * i + k
        return pos // 8, pos % 8
    j, i4, f = i // 16, (i % 16) // 4, i % 4   # high plane
    return d // 4 + 4 * (j // 2) + i4, 4 * (j % 2) + f


def pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint8)
    d = codes.shape[-1]
    if bits == 3 and d % 32:
        raise ValueError("3-bit rows need d a multiple of 32 (reading Z36)")
    nbytes = d * bits // 8
    out = np.zeros(codes.shape[:-1] + (nbytes,), dtype=np.uint8)
    for i in range(d):
        for k in range(bits):
            byte, bit_pos = _bit_position(i, k, bits, d)
            bit = (codes[..., i] >> k) & 1
            out[..., byte] |= (bit << bit_pos).astype(np.uint8)
    return out


def unpack_codes(packed: np.ndarray, bits: int, d: int) -> np.ndarray:
    packed = np.asarray(packed, dtype=np.uint8)
    out = np.zeros(packed.shape[:-1] + (d,), dtype=np.uint8)
    for i in range(d):
        for k in range(bits):
            byte, bit_pos = _bit_position(i, k, bits, d)
            bit = (packed[..., byte] >> bit_pos) & 1
            out[..., i] |= (bit << k).astype(np.uint8)
    return out


# ----------------------------------------------------------------------------------
# Paged cache format (reading Z24, DESIGN.md §5 "FORMAT"): pool[num_pages][H_kv][page_bytes];
# slot = page·P + offset u (P a multiple of 16).  One (page, kv-head) block =
#   K codes [P rows of rb = d·b/8 bytes] ‖ V codes [P·rb bytes] ‖ meta [P·(d/G)·8 bytes]
# padded to a multiple of 256 bytes.  The row bitstream (reading Z22) is unchanged; only
# the placement of whole rows / bytes inside the block is permuted for the decode kernel:
#   K row u   -> row position 16·(u//16) + 8·(u%2) + (u%16)//2   (even tokens of each
#                16-token tile first)
#   V byte j of row u -> 16·rb·(u//16) + 16·(32·(k//4) + 4·(j%8) + (u//4)%4) + 4·(k%4) + u%4
#                with k = j//8 (one 32-bit word = byte j of 4 consecutive tokens; words
#                grouped in 16-byte chunks so that the decode kernel's loads are
#                bank-conflict free)
#   meta of (u, group γ): chunk c = 128·(d/G)·(u//16) + 128·γ + 32·((u//4)%4);
#                fp16 (s_K, m_K) at c + 4·(u%4), fp16 (s_V, m_V) at c + 16 + 4·(u%4)
# ----------------------------------------------------------------------------------
@dataclass(frozen=True)
class PageFormat:
    d: int
    bits: int
    G: int
    P: int = 64

    @property
    def row_bytes(self) -> int:
        return self.d * self.bits // 8

    @property
    def kcodes_off(self) -> int:
        return 0

    @property
    def vcodes_off(self) -> int:
        return self.P * self.row_bytes

    @property
    def meta_off(self) -> int:
        return 2 * self.P * self.row_bytes

    @property
    def page_bytes(self) -> int:
        raw = 2 * self.P * self.row_bytes + self.P * (self.d // self.G) * 8
        return (raw + 255) // 256 * 256

    def krow_offset(self, u: int) -> int:
        """Offset (within the block) of K row u."""
        return self.kcodes_off + (16 * (u // 16) + 8 * (u % 2) + (u % 16) // 2) * self.row_bytes

    def vbyte_offsets(self, u: int) -> np.ndarray:
        """Offsets (within the block) of the row_bytes bytes of V row u."""
        rb = self.row_bytes
        j = np.arange(rb)
        k = j // 8
        lane = 4 * (j % 8) + (u // 4) % 4
        if self.bits != 3:          # b in {2, 4}: words in 16-byte chunks per lane
            word = 128 * (k // 4) + 4 * lane + k % 4
            return self.vcodes_off + 16 * rb * (u // 16) + 4 * word + u % 4
        # b = 3 (reading Z36): per 16-token tile, the low-plane bytes j < d/4 laid out exactly as
        # a 2-bit row's bytes (16·d/4 bytes), then the high-plane bytes (16·d/8 bytes): high byte
        # e = 4·m + i (m = e // 4, i = e % 4) of row u at 16·(4·i + (u // 4) % 4) + 4·m + u % 4
        # (one 16-byte chunk per (i, 4-token group): the high bits a decode lane needs for its
        # channels, 4 tokens per 32-bit word)
        lo = j < self.d // 4
        word_lo = 128 * (k // 4) + 4 * lane + k % 4
        off_lo = 4 * word_lo + u % 4
        e = j - self.d // 4
        m, i = e // 4, e % 4
        off_hi = 16 * (self.d // 4) + 16 * (4 * i + (u // 4) % 4) + 4 * m + u % 4
        return self.vcodes_off + 16 * rb * (u // 16) + np.where(lo, off_lo, off_hi)

    def meta_offsets(self, u: int, grp: int):
        """Offsets of the fp16 pairs (s_K, m_K) and (s_V, m_V) of (row u, group grp)."""
        ng = self.d // self.G
        c = self.meta_off + 128 * ng * (u // 16) + 128 * grp + 32 * ((u // 4) % 4)
        return c + 4 * (u % 4), c + 16 + 4 * (u % 4)


def quantize_rotated(Kr, Vr, slots, fmt: PageFormat, pool: np.ndarray, rho_k=1.0, rho_v=1.0):
    """QuantizeAndWrite (Alg. 1) on already-rotated rows Kr, Vr [T, H, d] fp32."""
    Kc = clip_rows(Kr, rho_k)
    Vc = clip_rows(Vr, rho_v)
    ck, sk, mk = quantize_rows(Kc, fmt.bits, fmt.G)
    cv, sv, mv = quantize_rows(Vc, fmt.bits, fmt.G)
    pk = pack_codes(ck, fmt.bits)
    pv = pack_codes(cv, fmt.bits)
    ng = fmt.d // fmt.G
    T, H, _ = Kc.shape
    for t in range(T):
        page, off = divmod(int(slots[t]), fmt.P)
        for h in range(H):
            blk = pool[page, h]
            rb = fmt.row_bytes
            ko = fmt.krow_offset(off)
            blk[ko: ko + rb] = pk[t, h]
            blk[fmt.vbyte_offsets(off)] = pv[t, h]
            for grp in range(ng):
                ko_, vo_ = fmt.meta_offsets(off, grp)
                blk[ko_: ko_ + 4] = np.array([sk[t, h, grp], mk[t, h, grp]], np.float16).view(np.uint8)
                blk[vo_: vo_ + 4] = np.array([sv[t, h, grp], mv[t, h, grp]], np.float16).view(np.uint8)
    return pool


def quantize_append(K, V, slots, R_K, R_V, fmt: PageFormat, pool, rho_k=1.0, rho_v=1.0):
    """Alg. 1 `Prefill` rotate-before-write + QuantizeAndWrite."""
    return quantize_rotated(rotate(K, R_K), rotate(V, R_V), slots, fmt, pool, rho_k, rho_v)


def read_codes(pool: np.ndarray, slots, head: int, fmt: PageFormat):
    """The stored codes and metadata of the given slots of one KV head: (K codes [T, d],
    V codes [T, d], meta fp16 [T, d/G, 4] = (s_K, m_K, s_V, m_V))."""
    slots = np.asarray(slots, dtype=np.int64)
    T = slots.shape[0]
    rb = fmt.row_bytes
    ng = fmt.d // fmt.G
    pk = np.zeros((T, rb), np.uint8)
    pv = np.zeros((T, rb), np.uint8)
    meta = np.zeros((T, ng * 8), np.uint8)
    for t in range(T):
        page, off = divmod(int(slots[t]), fmt.P)
        blk = pool[page, head]
        ko = fmt.krow_offset(off)
        pk[t] = blk[ko: ko + rb]
        pv[t] = blk[fmt.vbyte_offsets(off)]
        for grp in range(ng):
            ko_, vo_ = fmt.meta_offsets(off, grp)
            meta[t, grp * 8: grp * 8 + 4] = blk[ko_: ko_ + 4]
            meta[t, grp * 8 + 4: grp * 8 + 8] = blk[vo_: vo_ + 4]
    m = meta.view(np.float16).reshape(T, ng, 4)
    return unpack_codes(pk, fmt.bits, fmt.d), unpack_codes(pv, fmt.bits, fmt.d), m


def read_rows(pool: np.ndarray, slots, head: int, fmt: PageFormat):
    """DequantHistory (Alg. 1) for one KV head: rotated-frame K̂r, V̂r [T, d] fp64."""
    ck, cv, m = read_codes(pool, slots, head, fmt)
    Kh = dequantize_rows(ck, m[..., 0], m[..., 1], fmt.G)
    Vh = dequantize_rows(cv, m[..., 2], m[..., 3], fmt.G)
    return Kh, Vh


# ----------------------------------------------------------------------------------
# Decode attention in the rotated frame (north star; equal in exact arithmetic to
# Alg. 1, reading Z21):  q̃ = q R_K ; ℓ_t = scale · q̃ · k̂_t ;
# p = softmax(ℓ) ; õ = Σ p_t v̂_t ; o = õ R_Vᵀ.  Unmasked over the given rows (Z20).
# Returns (o [g, d], lse [g]) with lse = ln Σ_t exp(ℓ_t) (natural log).
# ----------------------------------------------------------------------------------
def attend_rows(q: np.ndarray, Khat_rot: np.ndarray, Vhat_rot: np.ndarray,
                R_K: np.ndarray, R_V: np.ndarray, scale: float):
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    R_K = np.asarray(R_K, dtype=np.float64)
    R_V = np.asarray(R_V, dtype=np.float64)
    if Khat_rot.shape[0] == 0:
        return np.zeros_like(q), np.full(q.shape[0], -np.inf)
    qr = q @ R_K
    logits = scale * (qr @ np.asarray(Khat_rot, np.float64).T)     # [g, T]
    mx = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - mx)
    l = e.sum(axis=1, keepdims=True)
    p = e / l
    o_rot = p @ np.asarray(Vhat_rot, np.float64)
    return o_rot @ R_V.T, (mx + np.log(l))[:, 0]


def _slots_of(page_table_row, seq_len, P):
    t = np.arange(seq_len, dtype=np.int64)
    return np.asarray(page_table_row, dtype=np.int64)[t // P] * P + t % P


def attend(q, page_table, seq_lens, pool, R_K, R_V, fmt: PageFormat, num_kv_heads: int,
           scale=None, seqs=None):
    """`attend(q) -> o` over the packed paged cache.  q [B, H_q, d] (bf16 values).
    Returns o [B, H_q, d] fp64 and lse [B, H_q].  `seqs` restricts to a subset of b."""
    q = np.asarray(q, dtype=np.float64)
    B, Hq, d = q.shape
    g = Hq // num_kv_heads
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    o = np.zeros((B, Hq, d), dtype=np.float64)
    lse = np.full((B, Hq), -np.inf)
    for b in (range(B) if seqs is None else seqs):
        slots = _slots_of(page_table[b], int(seq_lens[b]), fmt.P)
        for h in range(num_kv_heads):
            Kh, Vh = read_rows(pool, slots, h, fmt)
            ob, lb = attend_rows(q[b, h * g:(h + 1) * g], Kh, Vh, R_K[h], R_V[h], scale)
            o[b, h * g:(h + 1) * g] = ob
            lse[b, h * g:(h + 1) * g] = lb
    return o, lse


def attend_mixed(q, page_table, seq_lens, pool, seg_k, seg_v, seg_lens, R_K, R_V, fmt: PageFormat,
                 num_kv_heads: int, scale=None):
    """Mixed-precision decode attention (§4; Alg. 1 DecodeStep P:L1632-1635,
    NEXT-1): the logical cache is the bf16 tokens of the segment (sink + recent, raw rows,
    seg_k/seg_v [B][H_kv][cap][d], first seg_lens[b] valid) plus the INT2 history in the paged
    pool (first seq_lens[b] tokens of the page table).  Written in the original frame exactly as
    Alg. 1: K̂_hist = Q(K̃)R_Kᵀ, V̂_hist = Q(Ṽ)R_Vᵀ, K_all = Concat(sink, K̂_hist, recent),
    o = softmax(scale · q K_allᵀ) V_all (token order does not change the result).
    Returns (o [B, H_q, d] fp64, lse [B, H_q])."""
    q = np.asarray(q, dtype=np.float64)
    B, Hq, d = q.shape
    g = Hq // num_kv_heads
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    o = np.zeros((B, Hq, d))
    lse = np.full((B, Hq), -np.inf)
    for b in range(B):
        slots = _slots_of(page_table[b], int(seq_lens[b]), fmt.P)
        for h in range(num_kv_heads):
            Kh, Vh = read_rows(pool, slots, h, fmt)
            K_all = np.concatenate([Kh @ np.asarray(R_K[h], np.float64).T,
                                    np.asarray(seg_k[b, h, :seg_lens[b]], np.float64)])
            V_all = np.concatenate([Vh @ np.asarray(R_V[h], np.float64).T,
                                    np.asarray(seg_v[b, h, :seg_lens[b]], np.float64)])
            if K_all.shape[0] == 0:
                continue
            logits = scale * (q[b, h * g:(h + 1) * g] @ K_all.T)
            mx = logits.max(axis=1, keepdims=True)
            e = np.exp(logits - mx)
            l = e.sum(axis=1, keepdims=True)
            o[b, h * g:(h + 1) * g] = (e / l) @ V_all
            lse[b, h * g:(h + 1) * g] = (mx + np.log(l))[:, 0]
    return o, lse


def attend_alg1(q_row, Khat_rot, Vhat_rot, R_K, R_V, scale):
    """Alg. 1 DecodeStep form: rotate every history row back
    (K̂ = k̂ R_Kᵀ, V̂ = v̂ R_Vᵀ), then o = softmax(scale · q K̂ᵀ) V̂ — self-check only."""
    Khat = np.asarray(Khat_rot, np.float64) @ np.asarray(R_K, np.float64).T
    Vhat = np.asarray(Vhat_rot, np.float64) @ np.asarray(R_V, np.float64).T
    logits = scale * (np.atleast_2d(np.asarray(q_row, np.float64)) @ Khat.T)
    logits -= logits.max(axis=1, keepdims=True)
    p = np.exp(logits)
    p /= p.sum(axis=1, keepdims=True)
    return p @ Vhat


# Theorem 1: E = Σ_j (Q(x̃_j) - x̃_j)ᵀ(Q(x̃_j) - x̃_j) with the clip included
# in the residual.
def residual_cov(Xr: np.ndarray, Xhat_rot: np.ndarray) -> np.ndarray:
    e = np.asarray(Xhat_rot, np.float64) - np.asarray(Xr, np.float64)
    e = e.reshape(-1, e.shape[-1])
    return e.T @ e


# Worked-example statistic: per-group max - min of one row.
def group_ranges(row: np.ndarray, G: int) -> np.ndarray:
    r = np.asarray(row, dtype=np.float64).reshape(-1, G)
    return r.max(axis=1) - r.min(axis=1)


# §5.1 BPE accounting: (1 - f)(b + meta_bits/G) + 16 f,
# f = (sink + recent)/L.
def effective_bpe(bits: int, G: int, sink_recent: int = 0, L: int = 1, meta_bits: int = 32) -> float:
    if sink_recent and L <= sink_recent:
        raise ValueError("L must exceed sink+recent")
    f = sink_recent / L if sink_recent else 0.0
    return (1.0 - f) * (bits + meta_bits / G) + 16.0 * f


# ----------------------------------------------------------------------------------
# Alg. 1 `CalibrateClip` (outputs c_K, c_V by reading Z17).  The paper does not
# specify the procedure; reading Z34: exhaustive search over a grid
# of clip ratios for the frozen-error surrogates of Theorem 1 (App A.6):
#   L_K(rho) = tr(R_K^T C_Q R_K E_K(rho)),  E_K(rho) = sum_j e_j^T e_j,
#   e_j = Q(clip(k_j R_K, rho)) - k_j R_K         (App A.5 clip + quantize)
# and L_V with (R_V, C_S, V).  One ratio pair per layer: the grid entry minimizing the sum over
# KV heads (S:L190 per-layer default); ties go to the earlier grid entry.
# ----------------------------------------------------------------------------------
def clip_objectives(X: np.ndarray, R: np.ndarray, C: np.ndarray, grid, bits: int, G: int) -> np.ndarray:
    """X [N, d] raw rows of one KV head, R [d, d], C [d, d] covariance target.  Returns the
    surrogate tr(R^T C R E(rho)) for each rho of the grid (fp64)."""
    Xr = rotate(np.asarray(X)[:, None, :], np.asarray(R)[None])[:, 0]   # fp32 rotated rows
    M = np.asarray(R, np.float64).T @ np.asarray(C, np.float64) @ np.asarray(R, np.float64)
    out = np.zeros(len(grid))
    for i, rho in enumerate(grid):
        Xc = clip_rows(Xr, rho)
        codes, s16, m16 = quantize_rows(Xc, bits, G)
        e = dequantize_rows(codes, s16, m16, G) - Xr.astype(np.float64)
        E = e.T @ e                                       # frozen residual covariance
        out[i] = np.trace(M @ E)
    return out


def calibrate_clip(K, V, R_K, R_V, C_Q, C_S, grid, bits: int, G: int):
    """K, V [N, H_kv, d]; R_* [H_kv, d, d]; C_* [H_kv, d, d].  Returns (obj [H_kv, 2, n_grid],
    rho_K, rho_V)."""
    H = K.shape[1]
    obj = np.zeros((H, 2, len(grid)))
    for h in range(H):
        obj[h, 0] = clip_objectives(K[:, h], R_K[h], C_Q[h], grid, bits, G)
        obj[h, 1] = clip_objectives(V[:, h], R_V[h], C_S[h], grid, bits, G)
    tot = obj.sum(axis=0)
    return obj, float(grid[int(np.argmin(tot[0]))]), float(grid[int(np.argmin(tot[1]))])
