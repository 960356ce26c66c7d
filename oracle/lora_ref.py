"""CPU restatement of addonsim/lora.py — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the reference line by line (paths relative to
/root/reference/pkg/src/addonsim/):

* accumulate      <- lora.py:84-95   fp64 row-block accumulation, BLOCK_ROWS=128,
                                     one rounding into float32 per element
* merge           <- lora.py:98-104  shape check, duplicate guard, recorded scale
* unmerge         <- lora.py:107-114 recorded scale, sign -1, any order
* create_and_replace <- lora.py:132-144 (same accumulate -> bitwise equal to merge)
* stack           <- lora.py:147-160 down' = [d_i * f32(s_i)], up' = [u_i], scale 1.0

Pinned: tests/test_oracle.py checks these reproduce the sha256 of the
reference's own outputs (tests/golden/lora_golden.json, made by
tests/golden/make_golden.py importing the unmodified reference).
Also provides ``accumulate_bf16`` — the bf16-weight definition of parity
used for the serving dtype: bf16(ref_fp32(upcast inputs)).
"""

from __future__ import annotations

import numpy as np

BLOCK_ROWS = 128  # lora.py:27


class OracleValidationError(ValueError):
    pass


def check_shapes(weight: np.ndarray, down: np.ndarray, up: np.ndarray) -> None:
    """lora.py:75-81."""
    h1, h2 = weight.shape
    if down.shape[0] != h1 or up.shape[1] != h2:
        raise OracleValidationError(
            f"shape ({down.shape[0]}, {up.shape[1]}) does not match layer ({h1}, {h2})")
    if down.shape[1] != up.shape[0]:
        raise OracleValidationError("rank mismatch")


def accumulate(weight: np.ndarray, down: np.ndarray, up: np.ndarray, scale: float,
               sign: float) -> None:
    """In place: weight = f32(f64(weight) + (sign*scale) * (f64(down) @ f64(up))),
    computed over 128-row blocks exactly like lora.py:84-95."""
    down = np.asarray(down, dtype=np.float32)
    up = np.asarray(up, dtype=np.float32)
    up64 = up.astype(np.float64)                                   # :88
    h1 = weight.shape[0]
    for row in range(0, h1, BLOCK_ROWS):                           # :90
        stop = min(row + BLOCK_ROWS, h1)                           # :91
        block = down[row:stop].astype(np.float64) @ up64           # :92
        acc = weight[row:stop].astype(np.float64)                  # :93
        acc += (sign * scale) * block                              # :94
        weight[row:stop] = acc.astype(np.float32)                  # :95


class Layer:
    """BaseLayer (lora.py:58-72) reduced to what the oracle needs."""

    def __init__(self, weight: np.ndarray):
        self.weight = np.asarray(weight, dtype=np.float32)
        self.patched: list[tuple[str, float]] = []


def merge(layer: Layer, adapter_id: str, down, up, adapter_scale: float = 1.0,
          scale: float | None = None) -> None:
    """lora.py:98-104."""
    check_shapes(layer.weight, down, up)
    if any(i == adapter_id for i, _ in layer.patched):
        raise OracleValidationError("already merged")
    eff = adapter_scale if scale is None else scale
    accumulate(layer.weight, down, up, eff, 1.0)
    layer.patched.append((adapter_id, eff))


def unmerge(layer: Layer, adapter_id: str, down, up) -> None:
    """lora.py:107-114."""
    check_shapes(layer.weight, down, up)
    for i, (existing, s) in enumerate(layer.patched):
        if existing == adapter_id:
            accumulate(layer.weight, down, up, s, -1.0)
            del layer.patched[i]
            return
    raise OracleValidationError("not merged")


def create_and_replace(weight: np.ndarray, down, up, scale: float) -> tuple[np.ndarray, np.ndarray]:
    """lora.py:132-144: (base copy, effective weight)."""
    base = weight.copy()
    eff = weight.copy()
    accumulate(eff, down, up, scale, 1.0)
    return base, eff


def stack(adapters: list[tuple[np.ndarray, np.ndarray, float]]) -> tuple[np.ndarray, np.ndarray]:
    """lora.py:147-160 on (down, up, scale) triples -> (down', up'), scale 1.0."""
    if not adapters:
        raise OracleValidationError("stack_adapters needs at least one adapter")
    downs = [np.asarray(d, np.float32) * np.float32(s) for d, _, s in adapters]
    ups = [np.asarray(u, np.float32) for _, u, _ in adapters]
    return np.concatenate(downs, axis=1), np.concatenate(ups, axis=0)


def accumulate_bf16(weight_bf16_as_f32: np.ndarray, down: np.ndarray, up: np.ndarray,
                    scale: float, sign: float) -> np.ndarray:
    """Parity definition for bf16 serving weights: the fp32 reference on the
    upcast inputs, rounded once to bf16 (round-to-nearest-even).  Inputs are
    float32 arrays holding bf16-representable values; returns float32 holding
    bf16 values."""
    w = np.array(weight_bf16_as_f32, dtype=np.float32, copy=True)
    accumulate(w, down, up, scale, sign)
    return round_to_bf16(w)


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (ties to even), returned as float32."""
    u = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    r = ((u + rounding) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def bf16_ulp(a: np.ndarray) -> np.ndarray:
    """Spacing of bf16 numbers at |a| (8 significant bits)."""
    a = np.abs(np.asarray(a, dtype=np.float64))
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -126)))
    return 2.0 ** (e - 7)
