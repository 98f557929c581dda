"""One-off: copy the five printed 8x16 rows of the worked example (PAPER.md, appendix
`app:intuition_uhp`) into tests/golden/worked_example_layer10.txt.
Run here once; the fixture is committed and the tests never read /root/reference."""
import re, sys

SRC = "/root/reference/PAPER.md"
BLOCKS = [  # (name, first line, last line) of each printed array (1-based, inclusive)
    ("raw_K_t", 163, 171),          # K_{t,.} raw token
    ("K_UQ", 186, 194),             # (K U_Q)_{t,.}
    ("K_UQ_H", 209, 217),           # (K U_Q H_Had)_{t,.}
    ("K_UQ_H_P", 232, 240),         # (K U_Q H_Had P_K)_{t,.}
    ("K_H", 255, 263),              # (K H_Had)_{t,.}
]
lines = open(SRC).read().split("\n")
out = ["# Worked example, Qwen3-4B-Thinking layer 10, kv-head 0, token t=5 (PAPER.md appendix",
       "# 'Intuition of the combination R_K = U_Q H_Had P_K', printed to 2 decimals).",
       "# One row per printed 8x16 array, channel j = 16*gridrow + gridcol. Source lines:"]
for name, a, b in BLOCKS:
    vals = []
    for ln in lines[a - 1:b]:
        if "hline" in ln:
            continue
        ln = ln.replace("\\mathbf{", "").replace("}", "").replace("\\\\", "")
        vals += [float(v) for v in ln.split("&")]
    assert len(vals) == 128, (name, len(vals))
    out.append(f"# {name}: PAPER.md L{a}-L{b}")
    out.append(name + " " + " ".join(f"{v:.2f}" for v in vals))
open(sys.argv[1], "w").write("\n".join(out) + "\n")
