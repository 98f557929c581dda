"""Summarize an ncu report (raw metrics + per-SASS-line hot spots) for profiles/."""
import csv, io, subprocess, sys

rep = sys.argv[1]
kfilt = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []   # optional kernel-name regex
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + kfilt, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "sm__inst_executed.sum", "smsp__inst_executed.avg.per_cycle_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__warps_issue_stalled", "lts__t_bytes.sum"]
for i, h in enumerate(hdr):
    if any(h == w or (h.startswith(w) and w.endswith("stalled")) for w in want):
        print(f"{h} = {vals[i]} {rows[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kfilt,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0
keys = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(f(r, k) for r in data) for k in keys}
tot = sum(agg.values()) or 1
print("stall breakdown (% of samples):", ", ".join(f"{k[6:]}={100*v/tot:.1f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
print("instructions executed (warp-level):", sum(f(r, "Instructions Executed") for r in data))
print("top SASS lines by samples:")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:15]:
    st = sorted(((k[6:], f(r, k)) for k in keys), key=lambda x: -x[1])[:2]
    print(f"  {int(f(r,'Warp Stall Sampling (All Samples)')):5d} {r[ix['Source']].strip()[:60]:60s} {st}")
print("shared-memory excess wavefronts by line:")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:4]:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"  {r[ix['Source']].strip()[:60]:60s} excess={f(r,'L1 Wavefronts Shared Excessive'):.0f} total={f(r,'L1 Wavefronts Shared'):.0f}")
