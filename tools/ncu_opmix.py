"""Warp-level instruction mix per unit of work from an ncu report: python tools/ncu_opmix.py REP UNITS [regex]"""
import collections, csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
cnt = collections.Counter()
for r in data:
    try:
        n = float(r[ix["Instructions Executed"]])
    except ValueError:
        continue
    op = r[ix["Source"]].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    cnt[o.split(".")[0]] += n
tot = sum(cnt.values())
for o, n in cnt.most_common(45):
    print(f"{o:10s} {n / units:8.1f} {100 * n / tot:5.1f}%")
print("total per unit", tot / units)
