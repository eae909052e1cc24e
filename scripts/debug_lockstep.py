"""Diagnose lockstep id mismatches: re-run MULTI in lockstep and report the first event where
a device id diverges from the teacher-forced CPU oracle, with the step's composition."""
import json, sys, tempfile
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.forward import OracleModel, token_stream
from paper_2603_10342_b200.agsv import Agsv
from tests.test_engine_gpu import MULTI, _with_backend

cfg = _with_backend(MULTI, "lockstep")
if len(sys.argv) > 1:
    cfg["policy"] = sys.argv[1]
t = Agsv().run(cfg)
recs = [json.loads(x) for x in t.jsonl(tempfile.mkdtemp()).splitlines()]
om = OracleModel("tiny", seed=recs[0]["seed"], max_ctx=4096)
V = 4096
sess, expect, resumes, hist = {}, {}, {}, {}
bad = 0
for i, r in enumerate(recs):
    if r.get("rec") != "ev":
        continue
    if r["k"] in ("issue", "prefill_done", "step_done", "stream_done", "rebind"):
        hist.setdefault(r.get("s", -1), []).append((i, r["k"], {k: r[k] for k in r if k in ("req", "len", "q", "ctx", "prefix", "emit", "chunk_s", "chunk", "ids")}))
    if r["k"] == "prefill_done":
        s = r["s"]
        o = sess.setdefault(s, om.session())
        if r["req"] == "cold":
            toks = token_stream(recs[0]["seed"], f"tok/{s}/cold", r["len"], V)
        else:
            k = resumes.get(s, 0); resumes[s] = k + 1
            toks = token_stream(recs[0]["seed"], f"tok/{s}/resume/{k}", r["len"], V)
        expect[s] = o.forward(toks)
        print(f"ev{i} prefill_done s{s} {r['req']} len {r['len']} ctx {r['ctx']} prefix {r['prefix']} first_id {r.get('first_id')} oracle {expect[s][0]} oracle_len {sess[s].length}")
    elif r["k"] == "step_done":
        ids = r.get("ids", [])
        for s, tok in zip(r["emit"], ids):
            nid, lg = expect[s]
            if tok != nid:
                bad += 1
                if bad <= 3:
                    top = np.sort(lg)[-2:]
                    print(f"MISMATCH ev{i} s{s} dev {tok} oracle {nid} margin {top[1]-top[0]:.3f} step emit {r['emit']} chunk_s {r.get('chunk_s')} chunk {r.get('chunk')} oracle_len {sess[s].length}")
            expect[s] = sess[s].forward([tok])
print("mismatches", bad)
print("device", recs[-1].get("device"))
