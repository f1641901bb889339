"""Error classes of the drop-in (streamcut/errors.py:4-13).

When the reference package is importable its own classes are reused, so code
written against streamcut (``except streamcut.CapacityError``) keeps working
after the swap; otherwise identically named classes are defined here.
"""

try:  # pragma: no cover - depends on the environment
    from streamcut.errors import CapacityError, FormatError, StreamcutError  # type: ignore
except Exception:  # noqa: BLE001
    class StreamcutError(Exception):
        """Base class for all errors raised by this package."""

    class FormatError(StreamcutError):
        """Malformed or inconsistent input data (files, labels, parameters)."""

    class CapacityError(StreamcutError):
        """A partition capacity constraint cannot be satisfied."""


class DeviceError(StreamcutError):
    """A CUDA failure inside libgrem_b200.so (no CPU fallback exists)."""


__all__ = ["StreamcutError", "FormatError", "CapacityError", "DeviceError"]
