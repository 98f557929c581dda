"""CPU oracle for the OSCAR hot path (arXiv 2605.17757) — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 numpy transcription of what the paper computes, used to check the
CUDA library.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product package
``paper_2605_17757_b200`` never imports it and shares no code with it (no kernels,
headers, helpers, tables or constant generators); the seeded input generators live in
``paper_2605_17757_b200/synth.py``, which holds none of the method's arithmetic.

Citations: ``P:Lnnn`` = /root/reference/PAPER.md line nnn (with its section / equation /
algorithm); ``S:Lnnn`` = SPEC.md; ``Zn`` = the paper-gap readings listed in DESIGN.md §3.

Parity status:
  * every function is pinned by ``tests/test_oracle_pins.py`` except
  * ``calibrate`` eigenvectors elementwise — **parity unpinned** (non-unique R for near-
    degenerate spectra); GPU-vs-oracle calibration parity is checked
    through invariants instead (Weyl, residual, orthogonality, Lemma);
  * the worked-example *table* aggregates — **parity unpinned** (needs the
    paper's Qwen3 activations); only the printed single-token rows are pins.
"""
from .oscar_oracle import *  # noqa: F401,F403
