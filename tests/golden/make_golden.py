"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes:
  tests/golden/lora_golden.json  — sha256 of every reference LoRA output on
      the test_lora.py cases and on all 100 criterion-9 layers, plus the
      reference's measured worst errors and the tiny exact cases in full.
  tests/golden/lora_small.npz    — full inputs + reference outputs for a few
      small cases (so GPU tests compare the kernel against the reference's own
      numbers, not only the oracle's).
  tests/golden/plan_golden.json  — plan_lora_patch / plan_pipeline_patch /
      serial/parallel step latencies / StepModel on a grid of inputs.
The reference is imported from /root/reference/pkg/src (never copied).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from addonsim import lora as R  # noqa: E402
from addonsim import orchestrator as O  # noqa: E402
from addonsim.model import LatencyProfile  # noqa: E402

import cases  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def lora_golden():
    out = {"reference": "addonsim 0.1.0 lora.py", "numpy": np.__version__, "cases": {}, "criterion9": []}
    small = {}
    # tiny exact cases (test_lora.py:35-47)
    lay = R.BaseLayer(np.eye(2, dtype=np.float32))
    R.merge_in_place(lay, R.LowRankAdapter("tiny", np.array([[1.0], [0.0]]), np.array([[0.0, 2.0]]), 1.0))
    out["cases"]["small_exact"] = lay.weight.tolist()
    lay = R.BaseLayer(np.eye(2, dtype=np.float32))
    R.merge_in_place(lay, R.LowRankAdapter("tiny", np.array([[1.0], [0.0]]), np.array([[0.0, 2.0]]), 1.0),
                     scale=0.5)
    out["cases"]["scale_override"] = lay.weight.tolist()

    tc = cases.lora_test_cases()
    for name, (w, d, u, s) in tc.items():
        layer = R.BaseLayer(w.copy())
        ad = R.LowRankAdapter(name, d, u, s)
        R.merge_in_place(layer, ad)
        merged = layer.weight.copy()
        R.unmerge_in_place(layer, ad)
        out["cases"][name] = {"merged_sha": sha(merged), "unmerged_sha": sha(layer.weight),
                              "round_trip_max": float(np.abs(layer.weight - w).max())}
        if w.size <= 200 * 150:
            small[f"{name}__w"] = w
            small[f"{name}__down"] = d
            small[f"{name}__up"] = u
            small[f"{name}__scale"] = np.float64(s)
            small[f"{name}__merged"] = merged
    # stacking (test_lora.py:131-142)
    w, da, ua, sa = tc["stack_a"]
    _, db, ub, sb = tc["stack_b"]
    A, B = R.LowRankAdapter("a", da, ua, sa), R.LowRankAdapter("b", db, ub, sb)
    seq = R.BaseLayer(w.copy())
    R.merge_in_place(seq, A, scale=0.7)
    R.merge_in_place(seq, B, scale=0.3)
    st = R.stack_adapters("stack", [(A, 0.7), (B, 0.3)])
    comb = R.BaseLayer(w.copy())
    R.merge_in_place(comb, st)
    out["cases"]["stacking"] = {"sequential_sha": sha(seq.weight), "stacked_sha": sha(comb.weight),
                                "stack_down_sha": sha(st.down), "stack_up_sha": sha(st.up),
                                "linearity_max": float(np.abs(seq.weight - comb.weight).max())}
    small["stacking__sequential"] = seq.weight.copy()
    small["stacking__stacked"] = comb.weight.copy()

    worst = {"round_trip": 0.0, "equivalence": 0.0, "linearity": 0.0}
    for layer_case in cases.criterion9_layers():
        i = layer_case["i"]
        w = layer_case["weight"]
        d1, u1, s1 = layer_case["first"]
        d2, u2, s2 = layer_case["second"]
        a1 = R.LowRankAdapter(f"a{i}", d1, u1, s1)
        a2 = R.LowRankAdapter(f"b{i}", d2, u2, s2)
        layer = R.BaseLayer(w.copy())
        R.merge_in_place(layer, a1)
        merged = layer.weight.copy()
        R.unmerge_in_place(layer, a1)
        rt = layer.weight.copy()
        aug = R.create_and_replace(R.BaseLayer(w.copy()), a1)
        seq = R.BaseLayer(w.copy())
        R.merge_in_place(seq, a1, 0.7)
        R.merge_in_place(seq, a2, 0.3)
        stk = R.stack_adapters(f"s{i}", [(a1, 0.7), (a2, 0.3)])
        comb = R.BaseLayer(w.copy())
        R.merge_in_place(comb, stk)
        worst["round_trip"] = max(worst["round_trip"], float(np.abs(rt - w).max()))
        worst["equivalence"] = max(worst["equivalence"], float(np.abs(aug.effective_weight - merged).max()))
        worst["linearity"] = max(worst["linearity"], float(np.abs(seq.weight - comb.weight).max()))
        out["criterion9"].append({
            "shape": list(w.shape), "rank": int(d1.shape[1]), "rank2": int(d2.shape[1]),
            "merged_sha": sha(merged), "round_trip_sha": sha(rt),
            "create_replace_sha": sha(aug.effective_weight), "sequential_sha": sha(seq.weight),
            "stacked_sha": sha(comb.weight),
            "merged_sum": float(merged.astype(np.float64).sum()),
        })
        if i < 12 and w.size <= 40000:
            for k, v in (("w", w), ("d1", d1), ("u1", u1), ("merged", merged), ("sequential", seq.weight),
                         ("stacked", comb.weight)):
                small[f"c9_{i}__{k}"] = v
            small[f"c9_{i}__s1"] = np.float64(s1)
    out["criterion9_worst"] = worst
    return out, small


def plan_golden():
    out = {"plan_lora_patch": [], "plan_pipeline_patch": [], "step_latency": []}
    for load in [0.0, 1e-9, 10.0, 53.4, 53.4 * 3, 435.3125, 490.0, 1000.0, 2669.99, 2670.0, 10_000.0]:
        for step_ms in [53.4, 21.7, 9.5]:
            for steps in [1, 20, 30, 50]:
                p = O.plan_lora_patch(load, step_ms, 100.0, steps)
                out["plan_lora_patch"].append({"args": [load, step_ms, 100.0, steps],
                                               "boundary": p.patch_boundary_step,
                                               "first": p.first_patched_step,
                                               "delay": p.inserted_delay_ms})
    for loads in ([200.0, 400.0], [0.0, 0.0], [200.0, 10_000.0], [100.0, 200.0, 300.0, 400.0],
                  [435.3125], [5.0, 5.0, 5.0, 50.0]):
        for step_ms in [53.4, 9.5]:
            p = O.plan_pipeline_patch(loads, step_ms, 100.0, 30)
            out["plan_pipeline_patch"].append({
                "args": [loads, step_ms, 100.0, 30], "boundary": p.patch_boundary_step,
                "first": p.first_patched_step, "delay": p.inserted_delay_ms,
                "groups": [[g.load_complete_ms, g.boundary_step, g.patch_end_nominal_ms] for g in p.groups]})
    for frac in [0.4, 0.43923]:
        prof = LatencyProfile(encoder_mid_fraction=frac)
        for n in [1, 2, 3]:
            out["step_latency"].append({"fraction": frac, "n": n,
                                        "serial": O.serial_step_latency(n, prof),
                                        "parallel": O.parallel_step_latency(n, prof)})
    return out


def main():
    lg, small = lora_golden()
    (HERE / "lora_golden.json").write_text(json.dumps(lg, indent=1, sort_keys=True))
    np.savez_compressed(HERE / "lora_small.npz", **small)
    (HERE / "plan_golden.json").write_text(json.dumps(plan_golden(), indent=1, sort_keys=True))
    print("criterion-9 worst:", lg["criterion9_worst"])
    print("wrote", sorted(p.name for p in HERE.iterdir() if p.suffix in (".json", ".npz")))


if __name__ == "__main__":
    main()
