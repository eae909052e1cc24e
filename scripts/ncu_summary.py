"""Summarise ncu output for profiles/.

  python scripts/ncu_summary.py launches <launch-list.csv>      # per-kernel share of a launch list
  python scripts/ncu_summary.py full <report.ncu-rep> [...]      # key metrics of --set full captures

The launch list is the `--metrics gpu__time_duration.sum --clock-control none` pass: per-launch
times are cold-cache and serialised, so only each kernel's SHARE is comparable with bench.py.
"""
import collections
import csv
import gzip
import io
import json
import statistics
import subprocess
import sys


def _rows(text):
    hdr, out = None, []
    for r in csv.reader(io.StringIO(text)):
        if "Kernel Name" in r or "ID" in r[:1] and "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def _short(name):
    n = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return n.split("(")[0]


def launches(path):
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as f:
        text = f.read()
    data = [d for d in _rows(text) if d.get("Metric Name") == "gpu__time_duration.sum"]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}
    agg = collections.defaultdict(list)
    for d in data:
        agg[(_short(d["Kernel Name"]), d["Grid Size"])].append(float(d["Metric Value"].replace(",", "")) *
                                                               scale.get(d["Metric Unit"], 1e-3))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for (k, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "grid": g, "launches": len(v), "median_us": round(statistics.median(v), 2),
                    "total_us": round(sum(v), 1), "share": round(sum(v) / tot, 4)})
    by_k = collections.defaultdict(float)
    for o in out:
        by_k[o["kernel"]] += o["share"]
    return {"launches": len(data), "total_us": round(tot, 1),
            "share_by_kernel": {k: round(v, 4) for k, v in sorted(by_k.items(), key=lambda kv: -kv[1])},
            "by_kernel_grid": out}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "gpc__cycles_elapsed.max", "launch__grid_size", "launch__cluster_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": _short(d.get("Kernel Name", "")), "grid": d.get("Grid Size")}
        for k in KEYS:
            if k in d and d[k] != "":
                u = units[hdr.index(k)]
                rec[k] = f"{d[k]} {u}".strip()
        stalls = {k.split("stalled_")[1]: float(d[k]) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued") and d[k]}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        rec["top_stalls(pc samples)"] = dict(top)
        out.append(rec)
    return out


if __name__ == "__main__":
    mode, paths = sys.argv[1], sys.argv[2:]
    if mode == "launches":
        print(json.dumps(launches(paths[0]), indent=1))
    else:
        print(json.dumps({p.split("/")[-1]: full(p) for p in paths}, indent=1))
