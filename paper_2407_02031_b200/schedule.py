"""Step-loop semantics of the add-on path: where a LoRA patch lands on the
denoising step grid, and the per-step latency model that measured B200 stage
times are reported in.

Mirrors (same names, argument meaning and error behaviour):
* plan_lora_patch / plan_pipeline_patch / PatchPlan / GroupPatch
      <- addonsim/orchestrator.py:191-278
* serial_step_latency / parallel_step_latency
      <- addonsim/orchestrator.py:170-188
* LatencyProfile (+ validate / with_overrides), PROFILES, get_profile and the
  stage functions  <- addonsim/model.py:28-158

The pipeline (pipeline.py) uses ``plan_lora_patch`` to pick the boundary k at
which the side-stream patch is swapped in: steps 1..k run on the pristine
weights, steps k+1.. on the patched shadow weights — the reference's
``first_patched_step = k + 1`` (orchestrator.py:227-241, 698-719).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, fields, replace
from typing import Optional, Sequence

from .errors import ValidationError

MIB_PER_GIB = 1024.0
STEPS_LIMIT = 1000


@dataclass(frozen=True)
class LatencyProfile:
    """Stage durations for one GPU + model (model.py:28-111).  The default
    values are the reference's H800/SDXL constants; ``b200_profile`` in
    profile.py builds one from measured B200 stage times."""

    unet_total_ms: float = 2670.0
    steps_reference: int = 50
    encoder_mid_fraction: float = 0.4
    controlnet_factor: float = 1.1
    text_encoder_ms: float = 10.0
    vae_decode_ms: float = 120.0
    comm_payload_mib: float = 108.0
    link_gibps: float = 200.0
    link_latency_ms: float = 0.3
    remote_fetch_gibps: float = 0.78
    patch_inplace_ms: float = 100.0
    patch_create_replace_ms_per_100mib: float = 2000.0 * 100.0 / 384.0
    unet_opt_multiplier: float = 1.0 / 1.2
    unet_opt_submultipliers: tuple = (1.064, 1.06, 1.072)

    def validate(self) -> "LatencyProfile":
        for name in ("unet_total_ms", "link_gibps", "remote_fetch_gibps"):
            if not getattr(self, name) > 0:
                raise ValidationError(f"{name} must be positive, got {getattr(self, name)!r}")
        for name in ("text_encoder_ms", "vae_decode_ms", "comm_payload_mib", "link_latency_ms",
                     "patch_inplace_ms", "patch_create_replace_ms_per_100mib"):
            if getattr(self, name) < 0:
                raise ValidationError(f"{name} must be non-negative, got {getattr(self, name)!r}")
        if not 1 <= self.steps_reference <= STEPS_LIMIT:
            raise ValidationError(f"steps_reference must be in [1, {STEPS_LIMIT}], got {self.steps_reference}")
        if not 0.0 < self.encoder_mid_fraction < 1.0:
            raise ValidationError(f"encoder_mid_fraction must be in (0, 1), got {self.encoder_mid_fraction!r}")
        if self.controlnet_factor <= 0:
            raise ValidationError(f"controlnet_factor must be positive, got {self.controlnet_factor!r}")
        if self.unet_opt_multiplier <= 0 or self.unet_opt_multiplier > 1:
            raise ValidationError(f"unet_opt_multiplier must be in (0, 1], got {self.unet_opt_multiplier!r}")
        return self

    def with_overrides(self, **overrides) -> "LatencyProfile":
        known = {f.name for f in fields(self)}
        unknown = sorted(set(overrides) - known)
        if unknown:
            raise ValidationError(f"unknown profile field(s): {', '.join(unknown)}")
        return replace(self, **overrides).validate()


PROFILES = {"paper-h800-sdxl": LatencyProfile()}


def _register_measured() -> None:
    """Add the measured B200 profile (profiles/b200_sdxl_profile.json, written
    by ``python -m paper_2407_02031_b200.profile`` on a B200) when present."""
    try:
        from .profile import load
        prof = load()
    except Exception:   # a malformed file must not break the planner
        prof = None
    if prof is not None:
        PROFILES["b200-sdxl"] = prof


def get_profile(name: str) -> LatencyProfile:
    if name == "b200-sdxl" and name not in PROFILES:
        _register_measured()
    if name not in PROFILES:
        raise ValidationError(f"unknown profile {name!r}; available: {sorted(PROFILES)}")
    return PROFILES[name]


def step_duration(profile: LatencyProfile, steps: Optional[int] = None) -> float:
    """model.py:126-133 — per-step time; `steps` is validated only."""
    steps = profile.steps_reference if steps is None else steps
    if not 1 <= steps <= STEPS_LIMIT:
        raise ValidationError(f"steps must be in [1, {STEPS_LIMIT}], got {steps}")
    return profile.unet_total_ms / profile.steps_reference


def encoder_mid_ms(profile: LatencyProfile) -> float:
    return step_duration(profile) * profile.encoder_mid_fraction


def decoder_ms(profile: LatencyProfile) -> float:
    return step_duration(profile) - encoder_mid_ms(profile)


def controlnet_step_ms(profile: LatencyProfile) -> float:
    return profile.controlnet_factor * encoder_mid_ms(profile)


def comm_ms(profile: LatencyProfile) -> float:
    """model.py:151-158: link latency + payload / bandwidth."""
    if profile.link_gibps <= 0:
        raise ValidationError(f"link_gibps must be positive, got {profile.link_gibps!r}")
    if profile.comm_payload_mib < 0:
        raise ValidationError(f"comm_payload_mib must be non-negative, got {profile.comm_payload_mib!r}")
    return profile.link_latency_ms + profile.comm_payload_mib / (profile.link_gibps * MIB_PER_GIB) * 1000.0


def serial_step_latency(n_controlnets: int, profile: LatencyProfile) -> float:
    """orchestrator.py:170-178: ControlNets inline on the base GPU."""
    if n_controlnets < 0:
        raise ValidationError(f"n_controlnets must be >= 0, got {n_controlnets}")
    return n_controlnets * controlnet_step_ms(profile) + encoder_mid_ms(profile) + decoder_ms(profile)


def parallel_step_latency(n_controlnets: int, profile: LatencyProfile) -> float:
    """orchestrator.py:181-188: ControlNets as a service; the decoder starts at
    max(encoder end, last branch arrival)."""
    if n_controlnets < 1:
        raise ValidationError(f"n_controlnets must be >= 1, got {n_controlnets}")
    branch = controlnet_step_ms(profile) + comm_ms(profile)
    return max(encoder_mid_ms(profile), branch) + decoder_ms(profile)


@dataclass(frozen=True)
class GroupPatch:
    load_complete_ms: float
    boundary_step: int
    patch_end_nominal_ms: float


@dataclass(frozen=True)
class PatchPlan:
    """orchestrator.py:198-211.  first_patched_step == steps + 1 means never."""

    load_complete_ms: float
    patch_boundary_step: Optional[int]
    first_patched_step: int
    inserted_delay_ms: float
    groups: tuple = ()


def first_boundary(constraint_ms: float, step_ms: float) -> int:
    """Smallest k >= 0 with k*step_ms >= constraint_ms, robust to float noise
    at an exact boundary (orchestrator.py:214-224)."""
    if constraint_ms <= 0:
        return 0
    k = int(math.ceil(constraint_ms / step_ms))
    while k > 0 and (k - 1) * step_ms >= constraint_ms:
        k -= 1
    while k * step_ms < constraint_ms:
        k += 1
    return k


def _check_grid(step_ms: float, steps: int) -> None:
    if step_ms <= 0:
        raise ValidationError(f"step_ms must be positive, got {step_ms!r}")
    if steps < 1:
        raise ValidationError(f"steps must be >= 1, got {steps}")


def plan_lora_patch(load_complete_ms: float, step_ms: float, patch_ms: float, steps: int) -> PatchPlan:
    """orchestrator.py:227-241: the whole adapter patches at the first step
    boundary at or after its load completes; too late => never, no delay."""
    _check_grid(step_ms, steps)
    if patch_ms < 0 or load_complete_ms < 0:
        raise ValidationError("patch_ms and load_complete_ms must be >= 0")
    k = first_boundary(load_complete_ms, step_ms)
    if k >= steps:
        return PatchPlan(load_complete_ms, None, steps + 1, 0.0)
    return PatchPlan(load_complete_ms, k, k + 1, patch_ms)


def plan_pipeline_patch(group_loads_ms: Sequence[float], step_ms: float,
                        per_group_patch_ms: float, steps: int) -> PatchPlan:
    """orchestrator.py:244-278: group m patches at the first boundary at or
    after max(its load, end of group m-1's patch)."""
    if not group_loads_ms:
        raise ValidationError("group_loads_ms must not be empty")
    if any(later < earlier for earlier, later in zip(group_loads_ms, group_loads_ms[1:])):
        raise ValidationError("group load completions must be non-decreasing")
    _check_grid(step_ms, steps)
    groups = []
    prev_end = 0.0
    last_k = None
    for load in group_loads_ms:
        k = first_boundary(max(load, prev_end), step_ms)
        if k >= steps:
            break
        end = k * step_ms + per_group_patch_ms
        groups.append(GroupPatch(load, k, end))
        prev_end = end
        last_k = k
    complete = len(groups) == len(group_loads_ms)
    return PatchPlan(
        load_complete_ms=float(group_loads_ms[-1]),
        patch_boundary_step=last_k if complete else None,
        first_patched_step=(last_k + 1) if complete else steps + 1,
        inserted_delay_ms=per_group_patch_ms * len(groups),
        groups=tuple(groups),
    )
