"""Measured B200 ProfileBundles (profiles/b200_profile_*.json, written on the GPU box by
paper_2603_10342_b200.profile_measure) are valid agentsim-profile-v1 documents for both our
library and the reference's validator (profile.cpp:81-128: full grid, positive, non-decreasing),
and drive the reference's config-time calibration the same way in both."""
import json
from pathlib import Path

import pytest

from paper_2603_10342_b200.agsv import Agsv
from tests.ref_oracle import ref_api

ROOT = Path(__file__).resolve().parents[1]
PROFILES = sorted((ROOT / "profiles").glob("b200_profile_*.json"))


@pytest.mark.parametrize("path", PROFILES, ids=[p.stem for p in PROFILES])
def test_measured_profile_validates(path):
    doc = json.loads(path.read_text())
    meta = doc.pop("measured")
    assert meta["green_contexts"], "profile must come from real Green Context partitions"
    assert doc["total_sms"] == doc["granularity"] * len(doc["decode"])
    for ph in ("decode", "cold_prefill", "resume_prefill"):
        r = [p["tokens_per_second"] for p in doc[ph]]
        assert all(b >= a > 0 for a, b in zip(r, r[1:])), ph
    Agsv().profile_validate(doc)
    ref_api().profile_validate(doc)


@pytest.mark.parametrize("path", PROFILES, ids=[p.stem for p in PROFILES])
def test_measured_profile_calibration_matches_reference(path):
    doc = json.loads(path.read_text())
    doc.pop("measured")
    cfg = {"workload": {"paradigm": "react", "model": "qwen2.5-3b", "concurrency": 4, "steps_per_session": 2},
           "profile": {"inline": doc}, "policy": "agentserve", "seed": 13}
    mine = json.loads(Agsv().config(cfg).resolved())
    ref = json.loads(ref_api().config(cfg).resolved())
    assert mine == ref
