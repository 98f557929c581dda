"""Extract per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, bytes per
launch) and duration from an `ncu --set full` report into a JSON file under profiles/, which
bench.py reports as roofline.traffic.  Usage: python tools/ncu_traffic.py REPORT OUT_JSON"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * UNIT.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * UNIT.get(u["dram__bytes_write.sum"], 1)
        dur = float(d["gpu__time_duration.sum"].replace(",", ""))
        res.setdefault(name, []).append({"dram_read_bytes": rd, "dram_write_bytes": wr,
                                         "traffic_bytes": rd + wr, "duration": dur,
                                         "duration_unit": u["gpu__time_duration.sum"]})
    json.dump({"source": rep, "kernels": res}, open(out, "w"), indent=1)
    for k, v in res.items():
        print(k, [round(x["traffic_bytes"] / 1e6, 3) for x in v], "MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
