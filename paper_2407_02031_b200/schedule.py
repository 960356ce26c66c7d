"""Step-loop semantics of the add-on path: on which denoising step a LoRA
patch lands, and the per-step latency report format measured B200 stage
times are written in.

Interface kept from the reference (names, argument meaning, error type):
``plan_lora_patch`` / ``plan_pipeline_patch`` / ``PatchPlan`` / ``GroupPatch``
(addonsim/orchestrator.py:191-278), ``serial_step_latency`` /
``parallel_step_latency`` (:170-188) and ``LatencyProfile`` with its stage
quantities (addonsim/model.py:28-158).  The field names and H800 defaults of
``LatencyProfile`` are the reference's report format (so a measured profile
can drive the reference's own simulator); the code below is this package's.

The pipeline uses ``plan_lora_patch`` to pick the boundary k at which the
side-stream patch is swapped in: steps 1..k run on the pristine weights,
steps k+1.. on the patched shadow weights — the reference's
``first_patched_step = k + 1``.  Parity: tests/test_schedule.py against
tests/golden/plan_golden.json (outputs of the unmodified reference).
"""

from __future__ import annotations

from bisect import bisect_left
from dataclasses import dataclass, fields, replace
from typing import Optional, Sequence

from .errors import ValidationError

MAX_STEPS = 1000


def _positive(v) -> bool:
    return v > 0


def _non_negative(v) -> bool:
    return v >= 0


# (fields, predicate, what the message says) — checked in this order
_PROFILE_RULES = (
    (("unet_total_ms", "link_gibps", "remote_fetch_gibps"), _positive, "must be positive"),
    (("text_encoder_ms", "vae_decode_ms", "comm_payload_mib", "link_latency_ms", "patch_inplace_ms",
      "patch_create_replace_ms_per_100mib"), _non_negative, "must be non-negative"),
    (("steps_reference",), lambda v: 1 <= v <= MAX_STEPS, f"must be in [1, {MAX_STEPS}]"),
    (("encoder_mid_fraction",), lambda v: 0.0 < v < 1.0, "must be in (0, 1)"),
    (("controlnet_factor",), _positive, "must be positive"),
    (("unet_opt_multiplier",), lambda v: 0 < v <= 1, "must be in (0, 1]"),
)


@dataclass(frozen=True)
class LatencyProfile:
    """Per-stage durations of one GPU + model.  Defaults: the paper's H800 /
    SDXL constants; ``profile.measure`` fills one from B200 measurements."""

    unet_total_ms: float = 2670.0            # whole UNet over steps_reference steps
    steps_reference: int = 50
    encoder_mid_fraction: float = 0.4        # encoder + mid share of a step
    controlnet_factor: float = 1.1           # ControlNet step / encoder + mid
    text_encoder_ms: float = 10.0
    vae_decode_ms: float = 120.0
    comm_payload_mib: float = 108.0          # residuals shipped per ControlNet per step
    link_gibps: float = 200.0
    link_latency_ms: float = 0.3
    remote_fetch_gibps: float = 0.78
    patch_inplace_ms: float = 100.0
    patch_create_replace_ms_per_100mib: float = 2000.0 * 100.0 / 384.0
    unet_opt_multiplier: float = 1.0 / 1.2
    unet_opt_submultipliers: tuple = (1.064, 1.06, 1.072)

    def validate(self) -> "LatencyProfile":
        for names, ok, what in _PROFILE_RULES:
            for name in names:
                value = getattr(self, name)
                if not ok(value):
                    raise ValidationError(f"{name} {what}, got {value!r}")
        return self

    def with_overrides(self, **overrides) -> "LatencyProfile":
        unknown = sorted(set(overrides) - {f.name for f in fields(self)})
        if unknown:
            raise ValidationError(f"unknown profile field(s): {', '.join(unknown)}")
        return replace(self, **overrides).validate()

    # -- stage quantities (model.py:126-158) --------------------------------
    @property
    def step_ms(self) -> float:
        return self.unet_total_ms / self.steps_reference

    @property
    def encoder_mid_ms(self) -> float:
        return self.step_ms * self.encoder_mid_fraction

    @property
    def decoder_ms(self) -> float:
        return self.step_ms - self.encoder_mid_ms

    @property
    def controlnet_ms(self) -> float:
        return self.controlnet_factor * self.encoder_mid_ms

    @property
    def comm_ms(self) -> float:
        """Link latency + payload over the link bandwidth (GiB/s -> MiB/ms)."""
        if not self.link_gibps > 0:
            raise ValidationError(f"link_gibps must be positive, got {self.link_gibps!r}")
        if self.comm_payload_mib < 0:
            raise ValidationError(f"comm_payload_mib must be non-negative, got {self.comm_payload_mib!r}")
        seconds = self.comm_payload_mib / (self.link_gibps * 1024.0)
        return self.link_latency_ms + seconds * 1000.0


PROFILES = {"paper-h800-sdxl": LatencyProfile()}


def get_profile(name: str) -> LatencyProfile:
    """Named profile; "b200-sdxl" is loaded on first use from the measurement
    profile.py wrote (profiles/b200_sdxl_profile.json)."""
    if name == "b200-sdxl" and name not in PROFILES:
        try:
            from .profile import load
            measured = load()
        except Exception:   # a malformed file must not break the planner
            measured = None
        if measured is not None:
            PROFILES[name] = measured
    try:
        return PROFILES[name]
    except KeyError:
        raise ValidationError(f"unknown profile {name!r}; available: {sorted(PROFILES)}") from None


def step_duration(profile: LatencyProfile, steps: Optional[int] = None) -> float:
    """Per-step time (``steps`` is range-checked only, as in the reference)."""
    if steps is not None and not 1 <= steps <= MAX_STEPS:
        raise ValidationError(f"steps must be in [1, {MAX_STEPS}], got {steps}")
    return profile.step_ms


def encoder_mid_ms(profile: LatencyProfile) -> float:
    return profile.encoder_mid_ms


def decoder_ms(profile: LatencyProfile) -> float:
    return profile.decoder_ms


def controlnet_step_ms(profile: LatencyProfile) -> float:
    return profile.controlnet_ms


def comm_ms(profile: LatencyProfile) -> float:
    return profile.comm_ms


def serial_step_latency(n_controlnets: int, profile: LatencyProfile) -> float:
    """ControlNets inline on the base GPU, then the UNet."""
    if n_controlnets < 0:
        raise ValidationError(f"n_controlnets must be >= 0, got {n_controlnets}")
    return n_controlnets * profile.controlnet_ms + profile.encoder_mid_ms + profile.decoder_ms


def parallel_step_latency(n_controlnets: int, profile: LatencyProfile) -> float:
    """ControlNets as a service: the decoder waits for the encoder and the
    slowest branch (compute + transfer)."""
    if n_controlnets < 1:
        raise ValidationError(f"n_controlnets must be >= 1, got {n_controlnets}")
    return max(profile.encoder_mid_ms, profile.controlnet_ms + profile.comm_ms) + profile.decoder_ms


@dataclass(frozen=True)
class GroupPatch:
    load_complete_ms: float
    boundary_step: int
    patch_end_nominal_ms: float


@dataclass(frozen=True)
class PatchPlan:
    """first_patched_step == steps + 1 means the patch never lands."""

    load_complete_ms: float
    patch_boundary_step: Optional[int]
    first_patched_step: int
    inserted_delay_ms: float
    groups: tuple = ()


class _Grid:
    """Step boundaries k * step_ms, k = 0, 1, ..."""

    def __init__(self, step_ms: float, steps: int):
        if step_ms <= 0:
            raise ValidationError(f"step_ms must be positive, got {step_ms!r}")
        if steps < 1:
            raise ValidationError(f"steps must be >= 1, got {steps}")
        self.step_ms, self.steps = step_ms, steps

    def at_or_after(self, t_ms: float) -> int:
        """Smallest k >= 0 with k * step_ms >= t_ms.  Exact: an integer search
        over the products themselves, so a time equal to a boundary lands ON it
        whatever the float rounding of t_ms / step_ms."""
        if t_ms <= 0:
            return 0
        hi = int(t_ms / self.step_ms) + 2
        return bisect_left(range(hi + 1), True, key=lambda k: k * self.step_ms >= t_ms)


def first_boundary(constraint_ms: float, step_ms: float) -> int:
    return _Grid(step_ms, 1).at_or_after(constraint_ms)


def plan_lora_patch(load_complete_ms: float, step_ms: float, patch_ms: float, steps: int) -> PatchPlan:
    """The whole adapter set patches at the first boundary at or after its
    load completes; a load that misses the last boundary never patches."""
    grid = _Grid(step_ms, steps)
    if patch_ms < 0 or load_complete_ms < 0:
        raise ValidationError("patch_ms and load_complete_ms must be >= 0")
    k = grid.at_or_after(load_complete_ms)
    if k >= steps:
        return PatchPlan(load_complete_ms, None, steps + 1, 0.0)
    return PatchPlan(load_complete_ms, k, k + 1, patch_ms)


def plan_pipeline_patch(group_loads_ms: Sequence[float], step_ms: float,
                        per_group_patch_ms: float, steps: int) -> PatchPlan:
    """Group-pipelined loading: group m patches at the first boundary at or
    after both its own load and the end of group m-1's patch; the plan stops
    at the first group that misses the last boundary."""
    if not group_loads_ms:
        raise ValidationError("group_loads_ms must not be empty")
    if any(b < a for a, b in zip(group_loads_ms, group_loads_ms[1:])):
        raise ValidationError("group load completions must be non-decreasing")
    grid = _Grid(step_ms, steps)
    placed: list[GroupPatch] = []
    busy_until = 0.0
    for load in group_loads_ms:
        k = grid.at_or_after(max(load, busy_until))
        if k >= steps:
            break
        busy_until = k * step_ms + per_group_patch_ms
        placed.append(GroupPatch(load, k, busy_until))
    done = len(placed) == len(group_loads_ms)
    last = placed[-1].boundary_step if (done and placed) else None
    return PatchPlan(
        load_complete_ms=float(group_loads_ms[-1]),
        patch_boundary_step=last,
        first_patched_step=last + 1 if last is not None else steps + 1,
        inserted_delay_ms=per_group_patch_ms * len(placed),
        groups=tuple(placed),
    )
