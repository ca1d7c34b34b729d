"""Add a per-cycle DRAM-traffic row to profiles/traffic.json from an ncu launch list.

usage: python tools/cycle_traffic.py LAUNCHES.csv NX NY NCYC [RELAX] [FUSED]

LAUNCHES.csv: `ncu --profile-from-start off --cache-control none --clock-control none
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`
of tools/profile_cycle.py with NCYC cycles.  Writes the mean over the cycles of the
summed dram read+write bytes of every kernel of one cycle (bench.py reads it as
roofline.cycle_dram_bytes, the north_star's "achieved HBM GB/s" of the whole cycle).
"""
import collections
import csv
import json
import os
import sys


def main():
    path, nx, ny, ncyc = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    relax = sys.argv[5] if len(sys.argv) > 5 else "point"
    fused = (sys.argv[6] != "0") if len(sys.argv) > 6 else True
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ix = {k: hdr.index(k) for k in ["ID", "Kernel Name", "Metric Name", "Metric Value"]}
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        d = per[int(r[ix["ID"]])]
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        d["name"] = r[ix["Kernel Name"]]
    ids = sorted(per)
    byts = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in ids)
    tns = sum(per[i].get("gpu__time_duration.sum", 0) for i in ids)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "profiles", "traffic.json")
    data = json.load(open(out)) if os.path.exists(out) else {"launches": []}
    cyc = [c for c in data.get("cycles", []) if not (c["nx"] == nx and c["ny"] == ny and c.get("relax") == relax
                                                   and c.get("fused", True) == fused)]
    cyc.append({"nx": nx, "ny": ny, "relax": relax, "fused": fused, "cycles": ncyc,
                "launches_per_cycle": len(ids) / ncyc, "dram_bytes_per_cycle": byts / ncyc,
                "serialised_kernel_ms_per_cycle": tns / ncyc / 1e6, "source": os.path.basename(path),
                "how": "ncu --cache-control none --clock-control none launch list, dram read+write summed over "
                       "every kernel of a cycle, mean over the cycles"})
    data["cycles"] = cyc
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(cyc[-1]))


if __name__ == "__main__":
    main()
