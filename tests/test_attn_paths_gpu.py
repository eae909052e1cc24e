"""Every split-KV merge path of paged decode attention against the CPU oracle.

The default split rule (decode_splits, csrc/decode_attn.cu) picks one path per shape; the
others stay reachable through runtime switches and must give the same
answer.  Each variant re-runs the head_dim-128 case of test_forward_matches_oracle (2500 /
1300-token contexts, GQA group 3) in a fresh process, because the switches are read once
per process:
  forced 3 splits       -> 3-CTA thread-block cluster, DSMEM merge (odd cluster size)
  no cluster, 16 splits -> fp32 partials merged by the grid's last-arriving CTA per row
  combine kernel        -> fp32 partials merged by decode_combine_kernel
  1 split               -> no merge at all on long contexts
  persistent            -> one-wave persistent grid walking (row, kv head, split) units, held-block
                           warp merge, last-arriver split merge incl. empty splits of ragged rows
the admitted-resume chunk of a decode step through prefill attention (ASB_CHUNK_AS_DECODE=0) or
as one decode item per token (=2) instead of its (token, head) columns packed 8 per decode item
(the default, every path above runs it), and both prefill-attention
decompositions: the default work-unit list (only long causal items
split, one wave) and the uniform grid.z split (ASB_PREFILL_UNITS=0, optionally forced to 3).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CASE = "tests/test_forward_gpu.py::test_forward_matches_oracle[hd128-prompt_lens2-6]"


@pytest.mark.parametrize("env", [
    {"ASB_DECODE_SPLITS": "3"},
    {"ASB_ATTN_NO_CLUSTER": "1", "ASB_DECODE_SPLITS": "16"},
    {"ASB_ATTN_COMBINE": "1", "ASB_ATTN_NO_CLUSTER": "1"},
    {"ASB_DECODE_MAX_SPLITS": "1"},
    {"ASB_PREFILL_UNITS": "0"},
    {"ASB_PREFILL_UNITS": "0", "ASB_PREFILL_SPLITS": "3"},
    {"ASB_DECODE_PERSIST": "1"},
    {"ASB_DECODE_PERSIST": "1", "ASB_DECODE_MAX_SPLITS": "1"},
    {"ASB_CHUNK_AS_DECODE": "0"},
    {"ASB_CHUNK_AS_DECODE": "2"},
    {"ASB_CHUNK_AS_DECODE": "2", "ASB_DECODE_PERSIST": "1"},
], ids=["cluster3", "last_arriver16", "combine", "single", "prefill_uniform", "prefill_uniform3", "persistent",
        "persistent_single", "chunk_as_prefill", "chunk_per_token", "chunk_per_token_persistent"])
def test_decode_attention_merge_paths(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", CASE],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "1 passed" in r.stdout


def test_gemm_pull_reduction_switch():
    """The DSMEM-load split-K reduction (ASB_GEMM_PULL_REDUCE=1, the A/B baseline of the bulk
    push) stays correct on the cluster cases."""
    e = dict(os.environ)
    e["ASB_GEMM_PULL_REDUCE"] = "1"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gemm_gpu.py", "-k", "3072-1024-1-5 or 1000-640-1-6 or 896-896-1-7 or 512-256-1-3"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "16 passed" in r.stdout, r.stdout[-500:]

