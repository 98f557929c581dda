"""paper_2605_17757_b200 — B200-native (sm_100a) hot path of OSCAR (arXiv 2605.17757).

    liboscar.so (csrc/, C ABI in include/oscar.h)    calibrate / quantize_append / attend
    binding.py                                       thin ctypes binding (same names)
    synth.py                                         seeded synthetic inputs (no method math)
    parallel.py                                      rank sharding + NCCL covariance all-reduce

The binding is imported lazily so that the input generators stay importable on a host
without the built library; any computing call imports it and fails loudly if
liboscar.so is missing (there is no CPU fallback).
"""
__all__ = ["Oscar", "Config", "OscarError", "version"]


def __getattr__(name):
    if name in __all__:
        from . import binding
        return getattr(binding, name)
    raise AttributeError(name)
