"""Patch-group split for group-pipelined patching (orchestrator.py:244-278):
host logic only (CPU)."""

import pytest
import torch

from paper_2407_02031_b200 import unet as U
from paper_2407_02031_b200.errors import ValidationError
from paper_2407_02031_b200.patcher import split_patch_groups


@pytest.fixture(scope="module")
def toy():
    return U.init_unet(U.TOY, torch.device("cpu"), torch.bfloat16, 0)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 8])
def test_split_is_an_ordered_balanced_partition(toy, m):
    groups = split_patch_groups(toy, m)
    names = [n for n, _ in toy.matrices]
    assert len(groups) == m
    flat = [n for n in names if any(n in g for g in groups)]
    assert flat == names and sum(len(g) for g in groups) == len(names)
    # contiguous runs of the UNet order
    idx = [next(i for i, g in enumerate(groups) if n in g) for n in names]
    assert idx == sorted(idx)
    # fused storages (q|k|v, k|v) never straddle two groups
    for members in toy.fused.values():
        assert len({idx[names.index(x)] for x in members}) == 1
    sizes = [sum(toy.t[n + ".weight"].numel() for n in g) for g in groups]
    total = sum(sizes)
    assert max(sizes) <= 1.6 * total / m


def test_split_rejects_zero(toy):
    with pytest.raises(ValidationError):
        split_patch_groups(toy, 0)


def test_split_sdxl_layout_on_meta():
    """SDXL-shaped inventory (794 matrices, layout only): groups stay
    contiguous, byte-balanced, and never split a fused q|k|v or k|v storage."""
    p = U.init_unet(U.SDXL, torch.device("meta"), torch.bfloat16, 0)
    assert len(p.matrices) == 794
    for m in (2, 4, 8):
        groups = split_patch_groups(p, m)
        assert len(groups) == m
        names = [n for n, _ in p.matrices]
        idx = {n: next(i for i, g in enumerate(groups) if n in g) for n in names}
        assert [idx[n] for n in names] == sorted(idx[n] for n in names)
        for members in p.fused.values():
            assert len({idx[x] for x in members}) == 1
        sizes = [sum(p.t[n + ".weight"].numel() for n in g) for g in groups]
        assert max(sizes) <= 1.25 * sum(sizes) / m


def test_patch_schedule_weight_sets():
    """caas.PatchSchedule: per-step weight set and the events each step waits for."""
    from paper_2407_02031_b200.caas import PatchSchedule

    class S:
        def __init__(self):
            self.waits = []

        def wait_event(self, e):
            self.waits.append(e)

    s = S()
    sch = PatchSchedule([1, 1, 3], ["e0", "e1", "e2"], steps=5)
    seen = [sch.weights_at(k, s) for k in range(1, 6)]
    assert seen == ["pristine", "pg2", "pg2", "patched", "patched"]
    assert s.waits == ["e0", "e1", "e2"] and sch.first_full == 4
    s2 = S()
    miss = PatchSchedule([2, None], ["a", "b"], steps=4)          # second group missed the request
    assert [miss.weights_at(k, s2) for k in range(1, 5)] == ["pristine", "pristine", "pg1", "pg1"]
    assert miss.first_full == 5
    miss.finish(s2)
    assert s2.waits == ["a", "b"]
    single = PatchSchedule([0], ["x"], steps=2)                    # one launch, boundary 0
    assert [single.weights_at(k, S()) for k in (1, 2)] == ["patched", "patched"]
