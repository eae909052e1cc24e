"""Host logic of the bench configurations: the wall-clock SLO / controller calibration from a
measured ProfileBundle (workloads.calibrate) and the run configs of C1-C5."""
import json

import pytest

from paper_2603_10342_b200 import workloads


def _profile(steps_ms, B=16, g=16, S=144):
    """A profile whose decode step at level L is steps_ms[L-1] at batch B."""
    dec = [{"sms": g * (i + 1), "tokens_per_second": 1000.0 * B / t} for i, t in enumerate(steps_ms)]
    return {"granularity": g, "total_sms": S, "decode": dec}, {"decode_batch": B, "decode_ctx": 3000}


def test_tau_and_thresholds_follow_the_full_device_step():
    prof, meas = _profile([8.6, 4.7, 4.1, 3.15, 3.15, 3.15, 3.15, 3.14, 3.14])
    c = workloads.calibrate(prof, meas)
    tau = 1.5 * 3.14
    assert c["slo"]["tau_tpot_ms"] == pytest.approx(tau, abs=1e-3)
    assert c["controller"]["theta_high_ms"] == pytest.approx(workloads.THETA_HIGH_FRAC * tau, abs=1e-3)
    assert c["controller"]["theta_low_ms"] == pytest.approx(workloads.THETA_LOW_FRAC * tau, abs=1e-3)
    assert c["controller"]["theta_low_ms"] < c["controller"]["theta_high_ms"] <= tau
    # phase-dependent theta_high: below tau once no cold prefill is queued, above theta_low
    nc = c["backend"]["theta_high_no_cold_ms"]
    assert nc == pytest.approx(workloads.THETA_HIGH_NO_COLD_FRAC * tau, abs=1e-3)
    assert nc == 0.0 or c["controller"]["theta_low_ms"] < nc < tau


def test_base_level_keeps_corun_headroom():
    # level 2 meets tau in isolation (4.70 <= 4.71) but not with the 10% co-run allowance
    prof, meas = _profile([8.6, 4.70, 4.1, 3.15, 3.15, 3.15, 3.15, 3.14, 3.14])
    c = workloads.calibrate(prof, meas)
    assert c["controller"]["r_base_slots"] == 3 == c["controller"]["initial_r_slots"]


def test_base_level_leaves_the_prefill_partition_a_slot():
    prof, meas = _profile([100.0] * 8 + [3.0])
    assert workloads.calibrate(prof, meas)["controller"]["r_base_slots"] == 8


@pytest.mark.parametrize("name", sorted(workloads.CONFIGS))
def test_run_configs(name):
    cfg = workloads.run_config(name, clock="wall")
    assert cfg["workload"]["concurrency"] == workloads.CONFIGS[name]["agents"]
    assert cfg["backend"]["prefill_unit_tokens"] == workloads.UNIT_TOKENS
    sh = workloads.run_config(name, clock="wall", n_shards=4, shard=2)
    assert sh["workload"]["concurrency"] == 4 * workloads.CONFIGS[name]["agents"]
    assert (sh["workload"]["shard_index"], sh["workload"]["shard_count"]) == (2, 4)
    v = workloads.run_config(name, clock="virtual")
    assert "backend" not in v
    json.dumps(cfg)


def test_controller_interval_is_sixteen_full_device_steps():
    prof, meas = _profile([8.6, 4.7, 4.1, 3.15, 3.15, 3.15, 3.15, 3.14, 3.14])
    assert workloads.calibrate(prof, meas)["controller"]["delta_t_ms"] == pytest.approx(workloads.CTRL_STEPS * 3.14, abs=0.1)


def _with_resume(prof, rate):
    prof = dict(prof)
    prof["resume_prefill"] = [{"sms": d["sms"], "tokens_per_second": rate} for d in prof["decode"]]
    return prof


def test_resume_budget_closes_when_a_chunk_step_misses_tau():
    prof, meas = _profile([8.6, 4.7, 4.1, 3.15, 3.15, 3.15, 3.15, 3.14, 3.14])
    # base level 3 (4.1 ms); a 16-token chunk at 13.8k tok/s adds 1.16 ms -> 5.8 ms > tau 4.71
    c = workloads.calibrate(_with_resume(prof, 13800.0), meas)["controller"]
    assert c["initial_b_tokens"] == 0 == c["b_min_tokens"]
    # a 0.16 ms chunk fits: the reference's budget defaults stay
    c = workloads.calibrate(_with_resume(prof, 100000.0), meas)["controller"]
    assert "initial_b_tokens" not in c and "b_min_tokens" not in c
