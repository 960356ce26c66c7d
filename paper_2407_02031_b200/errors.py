"""Exception taxonomy, mirroring addonsim/errors.py:8-29.

When the reference package (``addonsim``) is importable in the same process,
each class here also derives from the reference class of the same name, so a
caller that catches ``addonsim.errors.ValidationError`` around a drop-in call
keeps working.  Without it the classes stand alone (same names, same
hierarchy); nothing else in this package depends on the reference."""

from __future__ import annotations

try:   # the drop-in case: the reference installed beside this package
    from addonsim import errors as _ref
except Exception:   # noqa: BLE001 — absent (or broken) reference: standalone classes
    _ref = None


def _bases(name: str, *own: type) -> tuple:
    """(reference class, own bases...) — reference first for a consistent MRO;
    the bare ``Exception`` base is implied by the reference class."""
    ref = getattr(_ref, name, None) if _ref is not None else None
    if not isinstance(ref, type):
        return own
    return (ref,) + tuple(o for o in own if o is not Exception)


class AddonSimError(*_bases("AddonSimError", Exception)):
    """Base class for all errors raised by this package (errors.py:8-9)."""


class ValidationError(*_bases("ValidationError", AddonSimError)):
    """A value violates a documented precondition (errors.py:12-13)."""


class ConfigError(*_bases("ConfigError", AddonSimError)):
    """A configuration document is malformed (errors.py:16-17)."""


class SimulationError(*_bases("SimulationError", AddonSimError)):
    """A run failed an internal invariant (errors.py:28-29)."""


class DeviceError(AddonSimError):
    """No usable sm_100 CUDA device / the native library is missing.

    Not in the reference (which is CPU-only); raised instead of silently
    falling back to a CPU path."""
