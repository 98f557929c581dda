"""Rounding-boundary check of a GPU-written pool against the oracle (TEST INFRASTRUCTURE ONLY,
same import rules as the rest of ``oracle/``).

The GPU rotates in fp32 (tensor cores with a bf16 hi/lo split of R, or CUDA-core FMAs); the
oracle rotates in fp64 and rounds once (``rotate``).  The north star bounds the difference per
row: max|x̃_gpu − x̃_oracle| <= 1e-5·‖x̃‖ (reading Z26), checked by the rotation hook tests.
Given that bound, a code or a metadata value may legitimately differ from the oracle's only
where the oracle's pre-rounding value lies within the bound of a rounding boundary.  This
module checks EVERY differing (token, head, K|V, group) of a pool against that rule:

  * fp16 metadata (App A.5, readings Z2-Z4): s16 = fp16(s), s = (mx − mn)/q_max,
    and m16 = fp16(mn).  A differing value must be the adjacent fp16 number and the oracle's
    fp32 s (resp. mn) must lie within the bound (2ε/q_max for s, ε for mn) of the midpoint
    between the two fp16 values.
  * codes with equal metadata (reading Z4): |Δc| = 1 and the oracle's exact
    pre-round value t = RN(x − m16)·inv within ε·inv of the half-integer between the two codes.
  * codes of a group whose metadata differs: the GPU code must be a correct rounding, under the
    GPU's own (s16, m16), of some value within ε of the oracle's x̃: |c − clamp((x̃ − m)/s)| <=
    1/2 + ε/s.

ε = tol_rel·‖x̃_row‖ (+1 ulp of the largest |x̃| in the row for fp32 storage), doubled when
clipping is on (the nearest-rank τ moves by at most the same ε, and clamping is 1-Lipschitz).
No value of the GPU path is an input of the oracle here: the oracle's x̃, codes and metadata
are computed from the same seeded inputs; the GPU pool is only read and judged.
"""
from __future__ import annotations

import numpy as np

from .oscar_oracle import PageFormat, clip_rows, quantize_rows_detail, read_codes

__all__ = ["check_pool_flips"]


def _fp16_neighbours(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """True where fp16 a and b are adjacent representable numbers (or equal)."""
    ia = a.astype(np.float16).view(np.uint16).astype(np.int64)
    ib = b.astype(np.float16).view(np.uint16).astype(np.int64)
    # map sign-magnitude to a monotone integer line
    ma = np.where(ia & 0x8000, -(ia & 0x7FFF), ia)
    mb = np.where(ib & 0x8000, -(ib & 0x7FFF), ib)
    return np.abs(ma - mb) <= 1


def check_pool_flips(got: np.ndarray, Xrot: dict, slots, fmt: PageFormat, rho=(1.0, 1.0),
                     tol_rel: float = 1e-5, heads=None):
    """got: the GPU pool [pages][H][page_bytes]; Xrot: {"K": x̃_K, "V": x̃_V}, oracle rotated rows
    [T][H][d] fp32 (before clipping); slots [T].  Returns a dict of counts; raises
    AssertionError with the first unexplained difference."""
    slots = np.asarray(slots, np.int64)
    G, bits = fmt.G, fmt.bits
    qmax = float(2 ** bits - 1)
    H = Xrot["K"].shape[1]
    stats = {"groups": 0, "meta_flips": 0, "code_flips": 0, "groups_with_meta_flip": 0}
    for h in (range(H) if heads is None else heads):
        ck_g, cv_g, meta_g = read_codes(got, slots, h, fmt)
        for side, (cg, sidx, midx, r) in {"K": (ck_g, 0, 1, rho[0]), "V": (cv_g, 2, 3, rho[1])}.items():
            x_raw = np.asarray(Xrot[side][:, h], np.float32)
            x = clip_rows(x_raw, r)
            c_o, s16_o, m16_o, s32_o, t_o = quantize_rows_detail(x, bits, G)
            s16_g, m16_g = meta_g[..., sidx], meta_g[..., midx]
            T, d = x.shape
            ng = d // G
            eps = tol_rel * np.linalg.norm(x_raw.astype(np.float64), axis=1)
            eps = eps + np.abs(x_raw).max(axis=1).astype(np.float64) * 2.0 ** -23
            if r < 1.0:
                eps = 2 * eps
            xg = x.astype(np.float64).reshape(T, ng, G)
            cgg = cg.reshape(T, ng, G).astype(np.int64)
            cog = c_o.reshape(T, ng, G).astype(np.int64)
            tog = t_o.reshape(T, ng, G)
            mn_o = x.reshape(T, ng, G).min(axis=-1).astype(np.float64)
            stats["groups"] += T * ng
            for t_, gi in np.argwhere((s16_g != s16_o) | (m16_g != m16_o) |
                                      (cgg != cog).any(axis=-1)):
                e = eps[t_]
                where = f"{side} head {h} token {t_} group {gi}"
                sg, so = float(s16_g[t_, gi]), float(s16_o[t_, gi])
                mg, mo = float(m16_g[t_, gi]), float(m16_o[t_, gi])
                meta_diff = sg != so or mg != mo
                if sg != so:
                    assert _fp16_neighbours(np.float16(sg), np.float16(so)), f"{where}: s16 {sg} vs {so}"
                    mid = (sg + so) / 2
                    assert abs(float(s32_o[t_, gi]) - mid) <= 2 * e / qmax + 2.0 ** -20 * abs(mid), \
                        f"{where}: s16 flip {sg} vs {so} not at a boundary (s = {s32_o[t_, gi]})"
                    stats["meta_flips"] += 1
                if mg != mo:
                    assert _fp16_neighbours(np.float16(mg), np.float16(mo)), f"{where}: m16 {mg} vs {mo}"
                    mid = (mg + mo) / 2
                    assert abs(mn_o[t_, gi] - mid) <= e + 2.0 ** -22 * abs(mid), \
                        f"{where}: m16 flip {mg} vs {mo} not at a boundary (min = {mn_o[t_, gi]})"
                    stats["meta_flips"] += 1
                if meta_diff:
                    stats["groups_with_meta_flip"] += 1
                    # every GPU code must be a correct rounding under the GPU's own metadata
                    xs = xg[t_, gi]
                    if sg > 0:
                        tq = np.clip((xs - mg) / sg, 0.0, qmax)
                        bad = np.abs(cgg[t_, gi] - tq) > 0.5 + e / sg + 1e-6
                    else:
                        bad = cgg[t_, gi] != 0
                    assert not bad.any(), f"{where}: codes inconsistent with the GPU metadata"
                    continue
                for c in np.nonzero(cgg[t_, gi] != cog[t_, gi])[0]:
                    a, b = int(cgg[t_, gi, c]), int(cog[t_, gi, c])
                    assert abs(a - b) == 1, f"{where} ch {c}: code {a} vs {b}"
                    inv = 1.0 / so if so > 0 else 0.0
                    half = min(a, b) + 0.5
                    assert abs(tog[t_, gi, c] - half) <= e * inv + 1e-6 * max(1.0, abs(half)), \
                        f"{where} ch {c}: code {a} vs {b} not at a rounding boundary (t = {tog[t_, gi, c]})"
                    stats["code_flips"] += 1
    return stats
