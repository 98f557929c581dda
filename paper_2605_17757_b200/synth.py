"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

Holds NONE of the method's arithmetic (no rotation, quantization, packing or attention):
only random draws shaped like the paper's workloads (DESIGN.md §6 "input recipe"):

* Q per KV group: q = z · diag(sqrt(λ)) · W_hᵀ, λ_j ∝ j^-1.5 (λ1/λ̄ ≈ 50, cf. the printed
  "λ1/λ̄ ≈ 46.9"), W_h Haar per KV head, the g query heads share W_h.
* K: z ⊙ σ with σ_c = 1 except 4 random outlier channels per head with σ = 12 (cf. the
  printed -30.62 / 14.19 outliers).
* V: 0.25 z.   SV (C_S input): z · diag(sqrt(ν)) · W'ᵀ, ν_j ∝ j^-1.
* decode q: N(0, 2²) so that logits scale·q·k have std ≈ 2 (a "peaky" variant uses 8).
* All tensors are rounded to bf16 (round-to-nearest-even) — the cache's input dtype.

numpy generators (host, small/parity sizes) and torch generators (device, bench sizes)
follow the same recipe.
"""
from __future__ import annotations

import numpy as np

OUTLIER_CHANNELS = 4
OUTLIER_SIGMA = 12.0
V_SIGMA = 0.25


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float values to the nearest bf16 (ties to even); returns float32 holding them."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def haar(rng: np.random.Generator, d: int) -> np.ndarray:
    z = rng.standard_normal((d, d))
    q, r = np.linalg.qr(z)
    return q * np.sign(np.diag(r))[None, :]


def gen_queries(rng, N: int, Hq: int, Hkv: int, d: int, decay: float = 1.5) -> np.ndarray:
    g = Hq // Hkv
    lam = np.arange(1, d + 1, dtype=np.float64) ** (-decay)
    lam *= d / lam.sum()
    out = np.zeros((N, Hq, d), dtype=np.float64)
    for h in range(Hkv):
        W = haar(rng, d)
        for i in range(g):
            z = rng.standard_normal((N, d))
            out[:, h * g + i, :] = (z * np.sqrt(lam)) @ W.T
    return bf16_round(out)


def gen_keys(rng, T: int, Hkv: int, d: int) -> np.ndarray:
    out = np.zeros((T, Hkv, d), dtype=np.float64)
    for h in range(Hkv):
        sig = np.ones(d)
        sig[rng.choice(d, OUTLIER_CHANNELS, replace=False)] = OUTLIER_SIGMA
        out[:, h, :] = rng.standard_normal((T, d)) * sig
    return bf16_round(out)


def gen_values(rng, T: int, Hkv: int, d: int) -> np.ndarray:
    return bf16_round(V_SIGMA * rng.standard_normal((T, Hkv, d)))


def gen_sv(rng, N: int, Hq: int, d: int) -> np.ndarray:
    nu = np.arange(1, d + 1, dtype=np.float64) ** -1.0
    nu *= d / nu.sum()
    out = np.zeros((N, Hq, d))
    for i in range(Hq):
        W = haar(rng, d)
        out[:, i, :] = (rng.standard_normal((N, d)) * np.sqrt(nu)) @ W.T * V_SIGMA
    return bf16_round(out)


def gen_decode_q(rng, B: int, Hq: int, d: int, sigma: float = 2.0) -> np.ndarray:
    return bf16_round(sigma * rng.standard_normal((B, Hq, d)))


def gen_rotation(rng, Hkv: int, d: int) -> np.ndarray:
    """A random orthogonal R per head (fp32) — used where a test needs "some R" that is
    not the output of calibration (downstream parity feeds one R to both sides)."""
    return np.stack([haar(rng, d) for _ in range(Hkv)]).astype(np.float32)


def contiguous_page_table(B: int, max_pages: int, shuffle_rng=None) -> np.ndarray:
    """Sequence b owns pages [b·max_pages, (b+1)·max_pages), optionally in shuffled order."""
    pt = np.arange(B * max_pages, dtype=np.int32).reshape(B, max_pages)
    if shuffle_rng is not None:
        flat = pt.reshape(-1).copy()
        shuffle_rng.shuffle(flat)
        pt = flat.reshape(B, max_pages)
    return pt


def slots_for(page_table: np.ndarray, positions, P: int) -> np.ndarray:
    """Slot ids (page·P + offset) of positions [B, n] under a page table."""
    positions = np.asarray(positions, dtype=np.int64)
    b = np.arange(page_table.shape[0])[:, None]
    return page_table[b, positions // P].astype(np.int64) * P + positions % P


def random_pool(rng, num_pages: int, Hkv: int, page_bytes: int, meta_off: int,
                meta_entries: int) -> np.ndarray:
    """Random packed pool bytes for attention-only parity at full size: uniform codes and
    fp16 metadata (s ~ U[0.3, 2.5], m ~ U[-4, -0.5]) like a quantized N(0, 1) row."""
    pool = rng.integers(0, 256, size=(num_pages, Hkv, page_bytes), dtype=np.uint8)
    n = num_pages * Hkv * meta_entries
    meta = np.empty((n, 4), dtype=np.float16)
    meta[:, 0] = rng.uniform(0.3, 2.5, n)
    meta[:, 1] = rng.uniform(-4.0, -0.5, n)
    meta[:, 2] = rng.uniform(0.05, 0.6, n)
    meta[:, 3] = rng.uniform(-1.0, -0.1, n)
    mb = meta.view(np.uint8).reshape(num_pages, Hkv, meta_entries * 8)
    pool[:, :, meta_off:meta_off + meta_entries * 8] = mb
    return pool


# ---------------------------------------------------------------- torch (device) versions
def torch_queries(gen, N, Hq, Hkv, d, device, decay=1.5):
    import torch
    g = Hq // Hkv
    lam = torch.arange(1, d + 1, dtype=torch.float32, device=device) ** (-decay)
    lam = lam * (d / lam.sum())
    out = torch.empty((N, Hq, d), dtype=torch.bfloat16, device=device)
    for h in range(Hkv):
        W, _ = torch.linalg.qr(torch.randn(d, d, generator=gen, device=device))
        for i in range(g):
            z = torch.randn(N, d, generator=gen, device=device)
            out[:, h * g + i] = ((z * lam.sqrt()) @ W.T).to(torch.bfloat16)
    return out


def torch_sv(gen, N, Hq, d, device):
    import torch
    nu = torch.arange(1, d + 1, dtype=torch.float32, device=device) ** -1.0
    nu = nu * (d / nu.sum())
    out = torch.empty((N, Hq, d), dtype=torch.bfloat16, device=device)
    for i in range(Hq):
        W, _ = torch.linalg.qr(torch.randn(d, d, generator=gen, device=device))
        z = torch.randn(N, d, generator=gen, device=device)
        out[:, i] = ((z * nu.sqrt()) @ W.T * V_SIGMA).to(torch.bfloat16)
    return out


def torch_keys(gen, T, Hkv, d, device):
    import torch
    sig = torch.ones(Hkv, d, device=device)
    for h in range(Hkv):
        idx = torch.randperm(d, generator=gen, device=device)[:OUTLIER_CHANNELS]
        sig[h, idx] = OUTLIER_SIGMA
    return (torch.randn(T, Hkv, d, generator=gen, device=device) * sig).to(torch.bfloat16)


def torch_values(gen, T, Hkv, d, device):
    import torch
    return (V_SIGMA * torch.randn(T, Hkv, d, generator=gen, device=device)).to(torch.bfloat16)


def torch_decode_q(gen, B, Hq, d, device, sigma=2.0):
    import torch
    return (sigma * torch.randn(B, Hq, d, generator=gen, device=device)).to(torch.bfloat16)


def torch_rotation(gen, Hkv, d, device):
    import torch
    Rs = [torch.linalg.qr(torch.randn(d, d, generator=gen, device=device))[0] for _ in range(Hkv)]
    return torch.stack(Rs).to(torch.float32).contiguous()


def torch_random_pool(gen, num_pages, Hkv, page_bytes, meta_off, meta_entries, device):
    """Device version of `random_pool` (same value distributions)."""
    import torch
    pool = torch.randint(0, 256, (num_pages, Hkv, page_bytes), generator=gen, device=device,
                         dtype=torch.int32).to(torch.uint8)
    n = num_pages * Hkv * meta_entries
    u = torch.rand(n, 4, generator=gen, device=device)
    lo = torch.tensor([0.3, -4.0, 0.05, -1.0], device=device)
    hi = torch.tensor([2.5, -0.5, 0.6, -0.1], device=device)
    meta = (lo + (hi - lo) * u).to(torch.float16)
    pool[:, :, meta_off:meta_off + meta_entries * 8] = meta.view(torch.uint8).reshape(
        num_pages, Hkv, meta_entries * 8)
    return pool
