"""Run-to-run determinism of the device forward: every reduction (split-K over clusters or
workspaces, split-KV merges, warp merges) is fixed-order, so the same prompts and decode tokens
in fresh sessions must give bit-identical logits every time.  This caught a real ordering bug:
kernels launched with programmatic dependent launch directly after a thread-block-cluster
launch were not reliably ordered after its stores (launch.cuh: pdl_for_launch)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("model", ["llama3.2-3b", "qwen2.5-0.5b"])
def test_decode_forward_is_bit_identical_across_runs(model):
    r = subprocess.run([sys.executable, "scripts/determinism.py", model, "4", "4"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 mismatching steps" in r.stdout, r.stdout[-2000:]
