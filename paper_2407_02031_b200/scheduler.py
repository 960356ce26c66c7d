"""DDIM (eta = 0) noise schedule tables for the fused K4 step.

The reference has no scheduler arithmetic; conventions follow
the public Stable Diffusion configs: scaled-linear betas 0.00085 -> 0.012 over
1000 training steps, "leading" timestep spacing with steps_offset = 1,
set_alpha_to_one = False.  Everything is computed once per (steps, guidance)
on the host in float64 and uploaded as the [steps, 4] coefficient table K4
indexes with the device step counter.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TRAIN_STEPS = 1000
BETA_START = 0.00085
BETA_END = 0.012
STEPS_OFFSET = 1


def alphas_cumprod() -> np.ndarray:
    betas = np.linspace(BETA_START ** 0.5, BETA_END ** 0.5, TRAIN_STEPS, dtype=np.float64) ** 2
    return np.cumprod(1.0 - betas)


@dataclass(frozen=True)
class DDIMTables:
    timesteps: np.ndarray   # [steps] int, descending
    coef: np.ndarray        # [steps, 4] float32: a_t, a_prev, guidance, 0


def ddim_tables(steps: int, guidance: float) -> DDIMTables:
    if not 1 <= steps <= TRAIN_STEPS:
        raise ValueError(f"steps must be in [1, {TRAIN_STEPS}]")
    ac = alphas_cumprod()
    ratio = TRAIN_STEPS // steps
    ts = (np.arange(0, steps) * ratio).round()[::-1].astype(np.int64) + STEPS_OFFSET
    coef = np.zeros((steps, 4), dtype=np.float64)
    for i, t in enumerate(ts):
        prev = t - ratio
        coef[i, 0] = ac[t]
        coef[i, 1] = ac[prev] if prev >= 0 else ac[0]
        coef[i, 2] = guidance
    return DDIMTables(ts, coef.astype(np.float32))
