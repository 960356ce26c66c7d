"""Step-loop semantics (schedule.py) against the reference's own outputs
(tests/golden/plan_golden.json) and its test cases (test_orchestrator.py:111-215)."""

import json
from pathlib import Path

import pytest

from paper_2407_02031_b200 import schedule as S
from paper_2407_02031_b200.errors import ValidationError

GOLD = json.loads((Path(__file__).parent / "golden" / "plan_golden.json").read_text())


def test_plan_lora_patch_grid_matches_reference():
    for case in GOLD["plan_lora_patch"]:
        p = S.plan_lora_patch(*case["args"])
        assert (p.patch_boundary_step, p.first_patched_step, p.inserted_delay_ms) == \
            (case["boundary"], case["first"], case["delay"]), case


def test_plan_pipeline_patch_grid_matches_reference():
    for case in GOLD["plan_pipeline_patch"]:
        p = S.plan_pipeline_patch(*case["args"])
        assert p.patch_boundary_step == case["boundary"]
        assert p.first_patched_step == case["first"]
        assert p.inserted_delay_ms == case["delay"]
        assert [[g.load_complete_ms, g.boundary_step, g.patch_end_nominal_ms] for g in p.groups] == case["groups"]


def test_step_latency_matches_reference():
    for case in GOLD["step_latency"]:
        prof = S.LatencyProfile(encoder_mid_fraction=case["fraction"])
        assert S.serial_step_latency(case["n"], prof) == case["serial"]
        assert S.parallel_step_latency(case["n"], prof) == case["parallel"]


def test_reference_known_answers():
    # test_orchestrator.py:139-160, test_model.py:37-41
    p = S.plan_lora_patch(435.3125, 53.4, 100.0, 50)
    assert (p.patch_boundary_step, p.first_patched_step, p.inserted_delay_ms) == (9, 10, 100.0)
    assert S.plan_lora_patch(3 * 53.4, 53.4, 100.0, 50).patch_boundary_step == 3
    assert S.plan_lora_patch(10_000.0, 53.4, 100.0, 50).first_patched_step == 51
    assert S.comm_ms(S.LatencyProfile()) == 0.82734375
    prof = S.LatencyProfile()
    assert S.serial_step_latency(3, prof) == pytest.approx(3 * 23.496 + 53.4, abs=1e-9)
    plan = S.plan_pipeline_patch([0.0, 0.0], 53.4, 100.0, 50)
    assert [g.boundary_step for g in plan.groups] == [0, 2]


def test_validation_messages():
    with pytest.raises(ValidationError):
        S.plan_lora_patch(10.0, 0.0, 100.0, 50)
    with pytest.raises(ValidationError):
        S.plan_lora_patch(-1.0, 53.4, 100.0, 50)
    with pytest.raises(ValidationError, match="non-decreasing"):
        S.plan_pipeline_patch([400.0, 200.0], 53.4, 100.0, 50)
    with pytest.raises(ValidationError, match="empty"):
        S.plan_pipeline_patch([], 53.4, 100.0, 50)
    with pytest.raises(ValidationError, match="unknown profile field"):
        S.LatencyProfile().with_overrides(bogus=1)
    with pytest.raises(ValidationError):
        S.parallel_step_latency(0, S.LatencyProfile())
