"""Pin the CPU oracle (oracle/lora_ref.py) to the reference's own outputs:
bit-for-bit sha256 equality with tests/golden/lora_golden.json, which
tests/golden/make_golden.py produced by running the unmodified reference."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import cases
from oracle import lora_ref

GOLD = json.loads((Path(__file__).parent / "golden" / "lora_golden.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def test_tiny_exact_cases():
    w = np.eye(2, dtype=np.float32)
    lora_ref.accumulate(w, np.array([[1.0], [0.0]]), np.array([[0.0, 2.0]]), 1.0, 1.0)
    assert w.tolist() == GOLD["cases"]["small_exact"] == [[1.0, 2.0], [0.0, 1.0]]
    w = np.eye(2, dtype=np.float32)
    lora_ref.accumulate(w, np.array([[1.0], [0.0]]), np.array([[0.0, 2.0]]), 0.5, 1.0)
    assert w.tolist() == GOLD["cases"]["scale_override"]


@pytest.mark.parametrize("name", ["round_trip", "order_first", "order_second", "create_replace",
                                  "stack_a", "stack_b", "no_full_delta"])
def test_test_lora_cases_bitwise(name):
    w, d, u, s = cases.lora_test_cases()[name]
    layer = lora_ref.Layer(w.copy())
    lora_ref.merge(layer, name, d, u, s)
    assert sha(layer.weight) == GOLD["cases"][name]["merged_sha"]
    lora_ref.unmerge(layer, name, d, u)
    assert sha(layer.weight) == GOLD["cases"][name]["unmerged_sha"]


def test_stacking_bitwise():
    tc = cases.lora_test_cases()
    w, da, ua, sa = tc["stack_a"]
    _, db, ub, sb = tc["stack_b"]
    seq = lora_ref.Layer(w.copy())
    lora_ref.merge(seq, "a", da, ua, sa, scale=0.7)
    lora_ref.merge(seq, "b", db, ub, sb, scale=0.3)
    sd, su = lora_ref.stack([(da, ua, 0.7), (db, ub, 0.3)])
    comb = lora_ref.Layer(w.copy())
    lora_ref.merge(comb, "s", sd, su, 1.0)
    g = GOLD["cases"]["stacking"]
    assert sha(sd) == g["stack_down_sha"] and sha(su) == g["stack_up_sha"]
    assert sha(seq.weight) == g["sequential_sha"]
    assert sha(comb.weight) == g["stacked_sha"]


def test_criterion9_bitwise_and_gates():
    worst = {"round_trip": 0.0, "equivalence": 0.0, "linearity": 0.0}
    for case, gold in zip(cases.criterion9_layers(), GOLD["criterion9"]):
        w = case["weight"]
        d1, u1, s1 = case["first"]
        d2, u2, s2 = case["second"]
        assert list(w.shape) == gold["shape"] and d1.shape[1] == gold["rank"]
        layer = lora_ref.Layer(w.copy())
        lora_ref.merge(layer, "a", d1, u1, s1)
        merged = layer.weight.copy()
        assert sha(merged) == gold["merged_sha"]
        lora_ref.unmerge(layer, "a", d1, u1)
        assert sha(layer.weight) == gold["round_trip_sha"]
        _, eff = lora_ref.create_and_replace(w, d1, u1, s1)
        assert sha(eff) == gold["create_replace_sha"]
        seq = lora_ref.Layer(w.copy())
        lora_ref.merge(seq, "a", d1, u1, s1, 0.7)
        lora_ref.merge(seq, "b", d2, u2, s2, 0.3)
        assert sha(seq.weight) == gold["sequential_sha"]
        sd, su = lora_ref.stack([(d1, u1, 0.7), (d2, u2, 0.3)])
        comb = lora_ref.Layer(w.copy())
        lora_ref.merge(comb, "s", sd, su, 1.0)
        assert sha(comb.weight) == gold["stacked_sha"]
        worst["round_trip"] = max(worst["round_trip"], float(np.abs(layer.weight - w).max()))
        worst["equivalence"] = max(worst["equivalence"], float(np.abs(eff - merged).max()))
        worst["linearity"] = max(worst["linearity"], float(np.abs(seq.weight - comb.weight).max()))
    assert worst == GOLD["criterion9_worst"]
    assert worst["round_trip"] <= 1e-5 and worst["equivalence"] <= 1e-6 and worst["linearity"] <= 1e-5


def test_oracle_errors():
    layer = lora_ref.Layer(np.zeros((4, 4), np.float32))
    with pytest.raises(lora_ref.OracleValidationError, match="does not match layer"):
        lora_ref.merge(layer, "bad", np.zeros((3, 2), np.float32), np.zeros((2, 4), np.float32))
    with pytest.raises(lora_ref.OracleValidationError, match="not merged"):
        lora_ref.unmerge(layer, "x", np.zeros((4, 2), np.float32), np.zeros((2, 4), np.float32))


def test_bf16_rounding_helper():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 0.0], np.float32)
    r = lora_ref.round_to_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == np.float32(1.0078125)
    assert abs(r[3] - x[3]) <= lora_ref.bf16_ulp(x[3]) / 2
