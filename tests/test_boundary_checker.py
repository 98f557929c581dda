"""CPU tests of oracle/boundary.py, the rounding-boundary checker the GPU append tests use: a pool
built by the oracle from rows perturbed within the stated rotation bound passes, and pools with
an injected error that is not a boundary flip (a code off by one away from .5, a code off by
two, a metadata value off by more than one ulp) fail."""
import numpy as np
import pytest

import oracle as O
from oracle.boundary import check_pool_flips
from paper_2605_17757_b200 import synth


def _setup(bits=2, G=64, T=200, H=2, seed=5):
    rng = np.random.default_rng(seed)
    fmt = O.PageFormat(128, bits, G, 64)
    K, V = synth.gen_keys(rng, T, H, 128), synth.gen_values(rng, T, H, 128)
    RK, RV = synth.gen_rotation(rng, H, 128), synth.gen_rotation(rng, H, 128)
    slots = rng.permutation(4 * 64)[:T].astype(np.int64)
    rot = {"K": O.rotate(K, RK), "V": O.rotate(V, RV)}
    return rng, fmt, rot, slots


def _pool(fmt, rot, slots, npages=4):
    pool = np.zeros((npages, rot["K"].shape[1], fmt.page_bytes), np.uint8)
    O.quantize_rotated(rot["K"], rot["V"], slots, fmt, pool)
    return pool


@pytest.mark.parametrize("bits,G", [(2, 64), (3, 32), (4, 128)])
def test_perturbed_rotation_passes(bits, G):
    rng, fmt, rot, slots = _setup(bits, G)
    # a "GPU" whose rotation differs by up to 0.9e-5 of the row norm (within the stated bar)
    pert = {}
    for k, x in rot.items():
        n = np.linalg.norm(x.astype(np.float64), axis=-1, keepdims=True)
        pert[k] = (x + 0.9e-5 * n * rng.uniform(-1, 1, x.shape)).astype(np.float32)
    got = _pool(fmt, pert, slots)
    st = check_pool_flips(got, rot, slots, fmt)
    assert st["code_flips"] + st["meta_flips"] > 0           # the perturbation did flip something


def test_injected_errors_fail():
    rng, fmt, rot, slots = _setup()
    ref = _pool(fmt, rot, slots)
    check_pool_flips(ref, rot, slots, fmt)                     # identical pool: nothing to explain
    # (1) a K code changed by one far from a boundary
    c_o, s16, m16, _, t = O.quantize_rows_detail(rot["K"][:, 0], 2, 64)
    frac = np.abs(t - np.floor(t) - 0.5)
    r, c = np.unravel_index(np.argmax(frac * (c_o < 3)), frac.shape)
    bad = ref.copy()
    page, off = divmod(int(slots[r]), 64)
    ko = fmt.krow_offset(off) + (2 * c) // 8
    bad[page, 0, ko] ^= np.uint8(1 << ((2 * c) % 8))           # flips the low bit of code c
    with pytest.raises(AssertionError):
        check_pool_flips(bad, rot, slots, fmt)
    # (2) a metadata scale changed by several ulps
    bad = ref.copy()
    mo, _ = fmt.meta_offsets(off, 0)
    v = bad[page, 0, mo:mo + 2].view(np.uint16)
    bad[page, 0, mo:mo + 2] = (v + 5).view(np.uint8)
    with pytest.raises(AssertionError):
        check_pool_flips(bad, rot, slots, fmt)
