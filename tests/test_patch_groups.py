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
