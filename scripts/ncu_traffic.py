"""DRAM traffic per launch for the bench roofline (`traffic` key): reads an ncu CSV with
dram__bytes_read.sum / dram__bytes_write.sum per launch over the decode steps of one config's
shape (scripts/step_launches.py) and writes profiles/ncu_traffic_<config>.json with the mean
bytes per launch of each bench category, next to the algorithmic bytes of the same launches.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file t.csv \\
      python scripts/step_launches.py llama3.2-3b 16 3000 --level=0 --ncu
  python scripts/ncu_traffic.py t.csv --config c3 --model llama3.2-3b --rows 16 --ctx 3000
"""
import argparse
import collections
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle.forward import PRESETS  # noqa: E402  (model dimensions only)

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--config", default="c2")
ap.add_argument("--model", default="qwen2.5-0.5b")
ap.add_argument("--rows", type=int, default=2)
ap.add_argument("--ctx", type=int, default=2300)
ap.add_argument("--steps", type=int, default=2, help="decode steps the capture covers")
a = ap.parse_args()

m = PRESETS[a.model]
D, HQ, HKV, HD, FFN, V, L, T = m["d"], m["hq"], m["hkv"], m["hd"], m["ffn"], m["vocab"], m["layers"], a.rows
QKV = (HQ + 2 * HKV) * HD


def lin(n, k, t, out_b=2):  # decode-linear algorithmic bytes: weights + activations in + out
    return 2 * (n * k + t * k) + out_b * t * n


step_gemm = L * (lin(QKV, D, T) + lin(D, HQ * HD, T) + lin(2 * FFN, D, T) + lin(D, FFN, T)) + lin(V, D, T, 4)
step_attn = L * T * a.ctx * 2 * HKV * HD * 2  # every context token's K and V, per layer

rows = {}
hdr = None
for r in csv.reader(io.StringIO(Path(a.csv).read_text())):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = rows.setdefault(d["ID"], {"kernel": d["Kernel Name"], "grid": d["Grid Size"]})
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
cats = collections.defaultdict(list)
for e in rows.values():
    k = e["kernel"]
    b = e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    if ("gemm_tn" in k and ("<32," in k or "<64," in k)) or "dgemv" in k or "tgemv" in k:  # decode linears
        cats["decode_gemm"].append(b)
    elif "decode_attn" in k:
        cats["decode_attn"].append(b)
n_gemm = len(cats["decode_gemm"]) or 1
n_attn = len(cats["decode_attn"]) or 1
out = {"_how": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over {a.steps} decode steps of the "
               f"{a.config.upper()} shape ({a.model}, {T} rows, ctx {a.ctx}); mean DRAM bytes per launch",
       "_algorithmic_decode_gemm_per_launch": a.steps * step_gemm / n_gemm,
       "_algorithmic_decode_attn_per_launch": a.steps * step_attn / n_attn}
for k, v in cats.items():
    out[k] = sum(v) / len(v)
    out[f"_{k}_launches"] = len(v)
dst = ROOT / "profiles" / f"ncu_traffic_{a.config}.json"
dst.write_text(json.dumps(out, indent=1))
print(json.dumps(out, indent=1))
