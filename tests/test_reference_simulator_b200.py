"""the measured B200 stage times (profiles/b200_sdxl_profile.json,
written by ``python -m paper_2407_02031_b200.profile`` on a B200) drive the
UNMODIFIED reference simulator (imported from /root/reference, never copied)
so its own policies report B200 numbers.  Runs only where the reference is
mounted (the build container), and checks that our schedule.py restatement
agrees with the reference's arithmetic on the measured profile."""

import sys
from dataclasses import asdict
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def addonsim():
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import addonsim  # noqa: F401
    from addonsim import model, orchestrator
    return model, orchestrator


def test_measured_profile_through_reference_simulator(addonsim):
    model, orch = addonsim
    from paper_2407_02031_b200 import schedule as S
    ours = S.get_profile("b200-sdxl")
    ref_prof = model.LatencyProfile(**{k: v for k, v in asdict(ours).items()}).validate()
    steps = ours.steps_reference
    cluster = model.ClusterSpec(base_workers=1, controlnet_gpus=2, prewarm_worker_controlnets=True,
                                prewarm_service_controlnets=True)
    from addonsim.addons import AddonCatalog
    catalog = AddonCatalog(controlnets={"cn-000": 2500.0, "cn-001": 2500.0}, loras={})
    totals = {}
    for name in (orch.SERIAL_COLOCATED, orch.CAAS):
        req = model.Request(request_id=0, arrival_ms=0.0, controlnets=("cn-000", "cn-001"), loras=(),
                            steps=steps)
        _, bd = orch.execute(req, orch.Policy(name), cluster, ref_prof, catalog)
        totals[name] = bd.total_ms
    # the reference's step arithmetic == our restatement, on the measured profile
    assert orch.serial_step_latency(2, ref_prof) == S.serial_step_latency(2, ours)
    assert orch.parallel_step_latency(2, ref_prof) == S.parallel_step_latency(2, ours)
    denoise_serial = steps * S.serial_step_latency(2, ours)
    denoise_caas = steps * S.parallel_step_latency(2, ours)
    fixed = ref_prof.text_encoder_ms + ref_prof.vae_decode_ms
    assert totals[orch.SERIAL_COLOCATED] == pytest.approx(fixed + denoise_serial, abs=1e-6)
    assert totals[orch.CAAS] == pytest.approx(fixed + denoise_caas, abs=1e-6)
    print(f"reference simulator on measured B200 stages: serial {totals[orch.SERIAL_COLOCATED]:.1f} ms, "
          f"CaaS {totals[orch.CAAS]:.1f} ms (denoise {denoise_serial:.1f} -> {denoise_caas:.1f} ms)")
    assert denoise_caas < denoise_serial
