"""The INTEGRATION.md shim, exercised: the unmodified reference package
(addonsim, pip-installed into baseline/_ref) with its ``lora._accumulate``
replaced by ours — exactly the 3-line binding a maintainer would add — then
the REFERENCE's own merge_in_place / unmerge_in_place / create_and_replace /
stack_adapters run on the cases of its test_lora.py (tests/golden/cases.py
replays their generators; expected outputs are the reference's own,
tests/golden/lora_small.npz) and on acceptance criterion 9
(test_acceptance.py:341-391: round trip <= 1e-5, route equivalence <= 1e-6,
linearity <= 1e-5).  Its bookkeeping and error messages stay the
reference's; only the arithmetic runs on the B200."""

import sys
from pathlib import Path

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
GOLD = np.load(Path(__file__).parent / "golden" / "lora_small.npz")


@pytest.fixture(scope="module")
def ref_lora():
    if not (REF / "addonsim").exists():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    import addonsim.lora as rl
    from paper_2407_02031_b200.lora import _accumulate
    original = rl._accumulate
    rl._accumulate = _accumulate            # the INTEGRATION.md shim
    yield rl
    rl._accumulate = original


def test_reference_api_on_its_own_cases(ref_lora):
    rl = ref_lora
    for name in ("order_first", "order_second", "stack_a", "stack_b"):
        w, d, u, s = (GOLD[f"{name}__w"], GOLD[f"{name}__down"], GOLD[f"{name}__up"],
                      float(GOLD[f"{name}__scale"]))
        layer = rl.BaseLayer(w.copy())
        rl.merge_in_place(layer, rl.LowRankAdapter(name, d, u, s))
        assert np.abs(layer.weight - GOLD[f"{name}__merged"]).max() <= 1e-5
    # the 2x2 known answers and the reference's own error messages (test_lora.py:35-78)
    layer = rl.BaseLayer(np.eye(2, dtype=np.float32))
    ad = rl.LowRankAdapter("tiny", np.array([[1.0], [0.0]]), np.array([[0.0, 2.0]]))
    rl.merge_in_place(layer, ad)
    assert np.array_equal(layer.weight, np.array([[1.0, 2.0], [0.0, 1.0]], dtype=np.float32))
    with pytest.raises(Exception, match="already merged"):
        rl.merge_in_place(layer, ad)
    rl.unmerge_in_place(layer, ad)
    assert np.array_equal(layer.weight, np.eye(2, dtype=np.float32))
    with pytest.raises(Exception, match="not merged"):
        rl.unmerge_in_place(layer, ad)


def test_reference_criterion9_through_the_shim(ref_lora):
    rl = ref_lora
    worst = {"round_trip": 0.0, "equivalence": 0.0, "linearity": 0.0}
    for case in cases.criterion9_layers():
        i, w = case["i"], case["weight"]
        (d1, u1, s1), (d2, u2, s2) = case["first"], case["second"]
        a1, a2 = rl.LowRankAdapter(f"a{i}", d1, u1, s1), rl.LowRankAdapter(f"b{i}", d2, u2, s2)
        layer = rl.BaseLayer(w.copy())
        rl.merge_in_place(layer, a1)
        merged = layer.weight.copy()
        rl.unmerge_in_place(layer, a1)
        worst["round_trip"] = max(worst["round_trip"], float(np.abs(layer.weight - w).max()))
        aug = rl.create_and_replace(rl.BaseLayer(w.copy()), a1)
        worst["equivalence"] = max(worst["equivalence"], float(np.abs(aug.effective_weight - merged).max()))
        seq = rl.BaseLayer(w.copy())
        rl.merge_in_place(seq, a1, 0.7)
        rl.merge_in_place(seq, a2, 0.3)
        comb = rl.BaseLayer(w.copy())
        rl.merge_in_place(comb, rl.stack_adapters(f"s{i}", [(a1, 0.7), (a2, 0.3)]))
        worst["linearity"] = max(worst["linearity"], float(np.abs(seq.weight - comb.weight).max()))
    print("criterion 9, reference API + B200 _accumulate:", worst)
    assert worst["round_trip"] <= 1e-5
    assert worst["equivalence"] <= 1e-6
    assert worst["linearity"] <= 1e-5
