"""The north_star's bf16 latent gate (rel-L2 <= 1e-3 per step vs the fp32
oracle) against the oracle's own rounding floor (oracle/bf16_floor.py): a
bf16 rounding of ONE activation tensor — the UNet's final GroupNorm+SiLU
output — already moves the latents by more than 1e-3 on config 1, so the
device bf16 path is gated against the bf16 floor instead."""

from oracle import bf16_floor as B


def test_single_bf16_site_exceeds_the_1e3_gate():
    cfg, up, cps, req = B.toy_inputs()
    tab = B.floor_table(cfg, up, cps, req, which={"conv_norm_out only", "every site"})
    one, every = tab["conv_norm_out only"], tab["every site"]
    print("conv_norm_out only:", ["%.1e" % e for e in one])
    print("every site:", ["%.1e" % e for e in every])
    assert max(one) > 1e-3
    assert max(every) > max(one)
