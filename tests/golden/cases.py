"""Deterministic input generators shared by make_golden.py and the tests.

They replay the reference tests' own generators (numpy default_rng streams):
* ``lora_test_cases``  — /root/reference/pkg/tests/test_lora.py:24-33 + the
  seeds/shapes of each test there (:35-158)
* ``criterion9_layers`` — /root/reference/pkg/tests/test_acceptance.py:341-391
  (seed 209, 100 layers, h1,h2 in [8,512], r in [1,64], W~N(0,1),
  down~N(0,1)/sqrt(r), up~N(0,1), scale~U(0.1,1.5))
"""

from __future__ import annotations

import numpy as np


def random_layer_and_adapter(rng, h1, h2, rank, scale=None):
    """test_lora.py:24-33: returns (weight, down, up, scale)."""
    weight = rng.uniform(-1, 1, size=(h1, h2)).astype(np.float32)
    down = rng.uniform(-1, 1, size=(h1, rank)).astype(np.float32)
    up = rng.uniform(-1, 1, size=(rank, h2)).astype(np.float32)
    s = rng.uniform(0.1, 1.5) if scale is None else scale
    return weight, down, up, float(s)


def lora_test_cases():
    """Named random cases of test_lora.py, in the order the tests draw them."""
    cases = {}
    rng = np.random.default_rng(1)                      # test_merge_unmerge_round_trip
    cases["round_trip"] = random_layer_and_adapter(rng, 300, 200, 32)
    rng = np.random.default_rng(2)                      # test_round_trip_any_unmerge_order
    cases["order_first"] = random_layer_and_adapter(rng, 128, 96, 8)
    cases["order_second"] = random_layer_and_adapter(rng, 128, 96, 16)
    rng = np.random.default_rng(3)                      # test_create_and_replace_matches_merge_bitwise
    cases["create_replace"] = random_layer_and_adapter(rng, 256, 192, 24)
    rng = np.random.default_rng(5)                      # test_stacked_adapters_equal_sequential_merges
    cases["stack_a"] = random_layer_and_adapter(rng, 200, 150, 8)
    cases["stack_b"] = random_layer_and_adapter(rng, 200, 150, 12)
    rng = np.random.default_rng(6)                      # test_merge_does_not_materialize_full_delta
    cases["no_full_delta"] = random_layer_and_adapter(rng, 1024, 1024, 16)
    return cases


def criterion9_layers(n_layers: int = 100):
    """Yields dicts with weight, (down, up, scale) for adapter and second, as
    test_acceptance.py:341-391 draws them (same rng call order)."""
    rng = np.random.default_rng(209)
    for i in range(n_layers):
        h1 = int(rng.integers(8, 513))
        h2 = int(rng.integers(8, 513))
        rank = int(rng.integers(1, 65))
        weight = rng.standard_normal((h1, h2)).astype(np.float32)

        def draw(r):
            down = (rng.standard_normal((h1, r)) / np.sqrt(r)).astype(np.float32)
            up = rng.standard_normal((r, h2)).astype(np.float32)
            return down, up, float(rng.uniform(0.1, 1.5))

        first = draw(rank)
        second = draw(int(rng.integers(1, 65)))
        yield {"i": i, "weight": weight, "first": first, "second": second}
