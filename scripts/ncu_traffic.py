"""DRAM traffic per launch for the bench roofline (`traffic` key): reads an ncu CSV with
dram__bytes_read.sum / dram__bytes_write.sum per launch over decode steps of the C2 shape
(qwen2.5-0.5b, scripts/step_launches.py) and writes profiles/ncu_traffic.json with the mean
bytes per launch of each bench category, next to the algorithmic bytes of the same launches.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file t.csv \\
      python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=0 --ncu
  python scripts/ncu_traffic.py t.csv
"""
import collections
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
# qwen2.5-0.5b decode linears at T = 2 rows (bytes = 2(NK + TK) + 2TN; LM head fp32 out)
D, QKV, FFN, V, T = 896, 1152, 4864, 151936, 2
ALG = {"qkv": 2 * (QKV * D + T * D) + 2 * T * QKV, "o": 2 * (D * D + T * D) + 2 * T * D,
       "gate_up": 2 * (2 * FFN * D + T * D) + 2 * T * FFN, "down": 2 * (D * FFN + T * FFN) + 2 * T * D,
       "lm_head": 2 * (V * D + T * D) + 4 * T * V}

rows = {}
hdr = None
for r in csv.reader(io.StringIO(Path(sys.argv[1]).read_text())):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = d["ID"]
        e = rows.setdefault(key, {"kernel": d["Kernel Name"], "grid": d["Grid Size"]})
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
cats = collections.defaultdict(list)
for e in rows.values():
    k = e["kernel"]
    b = e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    if ("gemm_tn" in k and ("<32," in k or "<64," in k)) or "dgemv" in k:  # decode (swap / small-batch) linears
        cats["decode_gemm"].append(b)
    elif "decode_attn" in k:
        cats["decode_attn"].append(b)
out = {"_how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over 2 decode steps of the C2 shape "
               "(qwen2.5-0.5b, 2 rows, ctx 2300, whole device); mean DRAM bytes per launch",
       "_algorithmic_decode_gemm_per_launch": (24 * (ALG["qkv"] + ALG["o"] + ALG["gate_up"] + ALG["down"]) + ALG["lm_head"]) / 97,
       "_algorithmic_decode_attn_per_launch": T * 2300 * 2 * 64 * 2 * 2}
for k, v in cats.items():
    out[k] = sum(v) / len(v)
    out[f"_{k}_launches"] = len(v)
(ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out, indent=1))
