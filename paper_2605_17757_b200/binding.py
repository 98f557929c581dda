"""Thin ctypes binding of liboscar.so (include/oscar.h) — argument marshalling only.

Every computing call runs the library's sm_100a kernels on the tensors' device; there is no
CPU or PyTorch fallback: if the shared library is missing, importing this module raises.
Tensors are torch CUDA tensors (device memory, streams and process groups are PyTorch's).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
# OSCAR_LIB selects another build of the same library (A/B experiments: tools/ab_attend.sh)
LIB_PATH = os.environ.get("OSCAR_LIB") or os.path.join(_HERE, "liboscar.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "the OSCAR hot path has no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

OK, ERR_ARG, ERR_DIM, ERR_UNSUPPORTED, ERR_CUDA, ERR_CONVERGENCE = range(6)
EXPORTED = [
    "oscar_create", "oscar_destroy", "oscar_last_error", "oscar_version", "oscar_page_bytes",
    "oscar_calib_accumulate", "oscar_calib_finalize", "oscar_quantize_append",
    "oscar_attend_workspace_bytes", "oscar_attend", "oscar_attend_mixed", "oscar_rotate",
    "oscar_quantize_rotated", "oscar_rotate_fwht", "oscar_set_variant", "oscar_calib_clip", "oscar_calib_sv",
    "oscar_decode_step",
]


class OscarConfig(ctypes.Structure):
    _fields_ = [
        ("head_dim", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32), ("bits", ctypes.c_int32),
        ("group_size", ctypes.c_int32), ("page_size", ctypes.c_int32),
        ("clip_ratio_k", ctypes.c_float), ("clip_ratio_v", ctypes.c_float),
        ("softmax_scale", ctypes.c_float), ("attend_pages_per_split", ctypes.c_int32),
    ]


_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_sig = {
    "oscar_create": (_i32, [ctypes.POINTER(OscarConfig), ctypes.POINTER(_vp)]),
    "oscar_destroy": (None, [_vp]),
    "oscar_last_error": (ctypes.c_char_p, []),
    "oscar_version": (ctypes.c_char_p, []),
    "oscar_page_bytes": (_sz, [_vp]),
    "oscar_calib_accumulate": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "oscar_calib_finalize": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp]),
    "oscar_quantize_append": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "oscar_attend_workspace_bytes": (_sz, [_vp, _i32, _i32]),
    "oscar_attend": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp, _i32,
                            _vp, _vp]),
    "oscar_decode_step": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp,
                                 _i32, _vp, _vp]),
    "oscar_attend_mixed": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                  _vp, _sz, _vp, _i32, _vp, _vp]),
    "oscar_rotate": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "oscar_rotate_fwht": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "oscar_quantize_rotated": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "oscar_set_variant": (_i32, [_vp, _i32]),
    "oscar_calib_sv": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp]),
    "oscar_calib_clip": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_float), _i32, _vp,
                                _vp, _vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class OscarError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: status {status}: {_lib.oscar_last_error().decode()}")


def _check(st: int, where: str):
    if st != OK:
        raise OscarError(st, where)


def version() -> str:
    return _lib.oscar_version().decode()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


@dataclass
class Config:
    head_dim: int = 128
    num_q_heads: int = 32
    num_kv_heads: int = 8
    bits: int = 2
    group_size: int = 64
    page_size: int = 64
    clip_ratio_k: float = 1.0
    clip_ratio_v: float = 1.0
    softmax_scale: float = 0.0
    attend_pages_per_split: int = 0


class Oscar:
    """One oscar_ctx.  Methods mirror the C ABI names without the `oscar_` prefix."""

    def __init__(self, cfg: Config):
        self.cfg = cfg
        c = OscarConfig(cfg.head_dim, cfg.num_q_heads, cfg.num_kv_heads, cfg.bits, cfg.group_size,
                        cfg.page_size, cfg.clip_ratio_k, cfg.clip_ratio_v, cfg.softmax_scale,
                        cfg.attend_pages_per_split)
        h = _vp()
        _check(_lib.oscar_create(ctypes.byref(c), ctypes.byref(h)), "oscar_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "oscar_destroy", None) is not None:
            _lib.oscar_destroy(h)
        self._h = None

    # ---------------------------------------------------------------- layout
    def page_bytes(self) -> int:
        return int(_lib.oscar_page_bytes(self._h))

    def attend_workspace_bytes(self, B: int, max_pages: int) -> int:
        return int(_lib.oscar_attend_workspace_bytes(self._h, B, max_pages))

    def set_variant(self, variant: int):
        _check(_lib.oscar_set_variant(self._h, variant), "oscar_set_variant")

    # ---------------------------------------------------------------- calibrate
    def calib_accumulate(self, Q, SV, acc, stream=None):
        _check(_lib.oscar_calib_accumulate(self._h, _ptr(Q), _ptr(SV), Q.shape[0], _ptr(acc),
                                           _stream(stream)), "oscar_calib_accumulate")

    def calib_finalize(self, acc, n_mats, n_rows, R_K, R_V, evals=None, info=None, stream=None):
        _check(_lib.oscar_calib_finalize(self._h, _ptr(acc), n_mats, n_rows, _ptr(R_K), _ptr(R_V),
                                         _ptr(evals), _ptr(info), _stream(stream)),
               "oscar_calib_finalize")

    def calib_sv(self, Q, K, V, seq_starts, SV, stream=None):
        _check(_lib.oscar_calib_sv(self._h, _ptr(Q), _ptr(K), _ptr(V), _ptr(seq_starts), seq_starts.shape[0],
                                   Q.shape[0], _ptr(SV), _stream(stream)), "oscar_calib_sv")

    def calib_clip(self, K, V, R_K, R_V, acc, grid, obj=None, stream=None):
        """CalibrateClip (reading Z34): surrogate objectives obj [H_kv, 2, n_grid] (fp64, device)
        and the per-layer choice (rho_K, rho_V) the library selects (argmin over the grid of the
        sum over KV heads, first grid entry on ties).  Synchronizes to read the two indices."""
        import torch
        n = len(grid)
        if obj is None:
            obj = torch.empty((self.cfg.num_kv_heads, 2, n), dtype=torch.float64, device=K.device)
        choice = torch.empty(2, dtype=torch.int32, device=K.device)
        g = (ctypes.c_float * n)(*[float(x) for x in grid])
        _check(_lib.oscar_calib_clip(self._h, _ptr(K), _ptr(V), K.shape[0], _ptr(R_K), _ptr(R_V), _ptr(acc),
                                     g, n, _ptr(obj), _ptr(choice), _stream(stream)), "oscar_calib_clip")
        ik, iv = choice.tolist()
        return obj, float(grid[ik]), float(grid[iv])

    # ---------------------------------------------------------------- quantize_append
    def quantize_append(self, K, V, slots, R_K, R_V, pool, stream=None):
        _check(_lib.oscar_quantize_append(self._h, _ptr(K), _ptr(V), _ptr(slots), K.shape[0],
                                          _ptr(R_K), _ptr(R_V), _ptr(pool), _stream(stream)),
               "oscar_quantize_append")

    # ---------------------------------------------------------------- attend
    def attend(self, q, page_table, seq_lens, pool, R_K, R_V, workspace, out, lse=None,
               stream=None):
        import torch
        out_fp32 = 1 if out.dtype == torch.float32 else 0
        _check(_lib.oscar_attend(self._h, _ptr(q), _ptr(page_table), _ptr(seq_lens), q.shape[0],
                                 page_table.shape[1], _ptr(pool), _ptr(R_K), _ptr(R_V),
                                 _ptr(workspace), workspace.numel() * workspace.element_size(),
                                 _ptr(out), out_fp32, _ptr(lse), _stream(stream)), "oscar_attend")

    def decode_step(self, q, k_new, v_new, page_table, seq_lens, pool, R_K, R_V, workspace, out,
                    lse=None, stream=None):
        """Alg. 1 DecodeStep: quantize_append of (k_new, v_new) at position seq_lens[b]-1, then
        attend(q) over seq_lens[b] tokens (one fused prologue kernel + the attention kernels)."""
        import torch
        out_fp32 = 1 if out.dtype == torch.float32 else 0
        _check(_lib.oscar_decode_step(self._h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(page_table),
                                      _ptr(seq_lens), q.shape[0], page_table.shape[1], _ptr(pool), _ptr(R_K),
                                      _ptr(R_V), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                      _ptr(out), out_fp32, _ptr(lse), _stream(stream)), "oscar_decode_step")

    def attend_mixed(self, q, page_table, seq_lens, pool, R_K, R_V, seg_k, seg_v, seg_lens, workspace,
                     out, lse=None, stream=None):
        import torch
        out_fp32 = 1 if out.dtype == torch.float32 else 0
        _check(_lib.oscar_attend_mixed(self._h, _ptr(q), _ptr(page_table), _ptr(seq_lens), q.shape[0],
                                       page_table.shape[1], _ptr(pool), _ptr(R_K), _ptr(R_V), _ptr(seg_k),
                                       _ptr(seg_v), _ptr(seg_lens), seg_k.shape[2], _ptr(workspace),
                                       workspace.numel() * workspace.element_size(), _ptr(out), out_fp32,
                                       _ptr(lse), _stream(stream)), "oscar_attend_mixed")

    # ---------------------------------------------------------------- test hooks
    def rotate(self, X, R, Xrot, stream=None):
        _check(_lib.oscar_rotate(self._h, _ptr(X), _ptr(R), _ptr(Xrot), X.shape[0],
                                 _stream(stream)), "oscar_rotate")

    def rotate_fwht(self, X, U, Xrot, stream=None):
        _check(_lib.oscar_rotate_fwht(self._h, _ptr(X), _ptr(U), _ptr(Xrot), X.shape[0],
                                      _stream(stream)), "oscar_rotate_fwht")

    def quantize_rotated(self, Krot, Vrot, slots, pool, stream=None):
        _check(_lib.oscar_quantize_rotated(self._h, _ptr(Krot), _ptr(Vrot), _ptr(slots),
                                           Krot.shape[0], _ptr(pool), _stream(stream)),
               "oscar_quantize_rotated")


def raw_call(name: str, *args):
    """Direct access to an exported symbol (used by the ABI tests)."""
    return getattr(_lib, name)(*args)
