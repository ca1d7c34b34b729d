"""Write profiles/traffic.json (per-launch DRAM bytes for bench.py's roofline.traffic)
and a metrics summary from ncu --set full captures.

usage: python tools/traffic.py NX NY REPORT.ncu-rep [REPORT ...]
"""
import csv, io, json, os, re, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    for v in r[2:]:
        yield {k: v[h.index(k)] for k in ["Kernel Name"] + KEYS if k in h}


def short(name):
    m = re.match(r"void (k_fused_(?:down|up))<(\d+), (\d+),", name)
    return f"{m.group(1)}<{m.group(2)}, {m.group(3)}>" if m else name.split("(")[0]


def main():
    nx, ny = int(sys.argv[1]), int(sys.argv[2])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", "traffic.json")
    data = {"source": "ncu --set full --clock-control none, one launch per report (tools/traffic.py)",
            "launches": []}
    if os.path.exists(path):
        data = json.load(open(path))
    for rep in sys.argv[3:]:
        for d in rows(rep):
            k = short(d["Kernel Name"])
            data["launches"] = [x for x in data["launches"] if not (x["kernel"] == k and x["nx"] == nx and x["ny"] == ny)]
            data["launches"].append({"kernel": k, "nx": nx, "ny": ny, "report": os.path.basename(rep),
                                     "dram_bytes_read": int(float(d["dram__bytes_read.sum"])),
                                     "dram_bytes_write": int(float(d["dram__bytes_write.sum"])),
                                     "metrics": {kk: d[kk] for kk in KEYS if kk in d}})
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
