"""Drop-in API behaviour of paper_2407_02031_b200.lora mirroring
/root/reference/pkg/tests/test_lora.py.  Validation paths run on CPU; every
numeric path is @gpu (there is no CPU fallback — checked here too)."""

import numpy as np
import pytest
import torch

from paper_2407_02031_b200 import lora as L
from paper_2407_02031_b200.errors import DeviceError, ValidationError


def small_adapter(scale=1.0):
    return L.LowRankAdapter("tiny", np.array([[1.0], [0.0]]), np.array([[0.0, 2.0]]), scale)


def test_rank_and_shape_validation_cpu():
    layer = L.BaseLayer(np.zeros((4, 4), np.float32))
    bad = L.LowRankAdapter("bad", np.zeros((3, 2), np.float32), np.zeros((2, 4), np.float32))
    with pytest.raises(ValidationError, match="does not match layer"):
        L.merge_in_place(layer, bad)
    with pytest.raises(ValidationError, match="rank mismatch"):
        L.LowRankAdapter("worse", np.zeros((4, 2), np.float32), np.zeros((3, 4), np.float32))
    with pytest.raises(ValidationError, match="factors must be 2-d"):
        L.LowRankAdapter("flat", np.zeros(4, np.float32), np.zeros((1, 4), np.float32))
    with pytest.raises(ValidationError, match="not merged"):
        L.unmerge_in_place(L.BaseLayer(np.eye(2, dtype=np.float32)), small_adapter())
    with pytest.raises(ValidationError):
        L.stack_adapters("empty", [])
    with pytest.raises(ValidationError):
        L.bench_merge(repeats=0)


def test_stack_adapters_layout_cpu():
    a = L.LowRankAdapter("a", np.ones((3, 2), np.float32), np.ones((2, 5), np.float32), 0.1)
    b = L.LowRankAdapter("b", 2 * np.ones((3, 1), np.float32), np.ones((1, 5), np.float32), 0.2)
    s = L.stack_adapters("s", [(a, 0.7), (b, 0.3)])
    assert s.rank == 3 and s.scale == 1.0
    assert np.array_equal(s.down[:, :2], np.ones((3, 2), np.float32) * np.float32(0.7))
    assert np.array_equal(s.down[:, 2:], 2 * np.ones((3, 1), np.float32) * np.float32(0.3))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    layer = L.BaseLayer(np.eye(2, dtype=np.float32))
    with pytest.raises(DeviceError):
        L.merge_in_place(layer, small_adapter())
    assert layer.patched == [] and np.array_equal(layer.weight, np.eye(2, dtype=np.float32))


def test_footprint_accounting_cpu():
    w = np.zeros((8, 6), np.float32)
    a = L.LowRankAdapter("a", np.zeros((8, 2), np.float32), np.zeros((2, 6), np.float32))
    aug = L.AugmentedLayer(w.copy(), w.copy(), [(a, 1.0)])
    assert aug.nbytes == 2 * L.BaseLayer(w).nbytes + a.nbytes


def test_errors_derive_from_the_reference_when_installed():
    """With the reference importable (baseline/_ref, the drop-in setting), a
    caller catching addonsim.errors.ValidationError catches ours too."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    ref = root / "baseline" / "_ref"
    if not (ref / "addonsim").exists():
        pytest.skip("reference not installed in baseline/_ref")
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import addonsim.errors as A\n"
            "from paper_2407_02031_b200 import errors as E\n"
            "assert issubclass(E.ValidationError, A.ValidationError)\n"
            "assert issubclass(E.ValidationError, E.AddonSimError)\n"
            "assert issubclass(E.AddonSimError, A.AddonSimError)\n"
            "try:\n    raise E.ValidationError('rank mismatch')\n"
            "except A.ValidationError as e:\n    print('caught', e)\n") % (str(ref), str(root))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "caught rank mismatch" in out.stdout
