"""Exception taxonomy, mirroring addonsim/errors.py:8-29 so callers that catch
the reference's ``ValidationError`` keep working against the drop-in."""


class AddonSimError(Exception):
    """Base class for all errors raised by this package (errors.py:8-9)."""


class ValidationError(AddonSimError):
    """A value violates a documented precondition (errors.py:12-13)."""


class ConfigError(AddonSimError):
    """A configuration document is malformed (errors.py:16-17)."""


class SimulationError(AddonSimError):
    """A run failed an internal invariant (errors.py:28-29)."""


class DeviceError(AddonSimError):
    """No usable sm_100 CUDA device / the native library is missing.

    Not in the reference (which is CPU-only); raised instead of silently
    falling back to a CPU path."""
