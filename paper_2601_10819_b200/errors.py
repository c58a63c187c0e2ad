"""Exception taxonomy of the reference (mvtrack3d/errors.py:10-46) for the
hot path, plus the mapping from C-ABI status codes back to it."""

from __future__ import annotations

from . import _lib as L


class BehindCamera(ValueError):
    """A point projects to non-positive depth in the camera frame."""


class OffsetOutOfRange(ValueError):
    """A learned keypoint offset component left the unit cube [-1, 1]."""


class NonFiniteWeight(ValueError):
    """A sampling plan contains a NaN or infinite weight or coordinate."""


class OddChannelCount(ValueError):
    """Feature channel count is odd; the packed-pair path needs pairs."""


class ChannelMismatch(ValueError):
    """Pyramid channel count does not match the query descriptor length."""


class AllOccluded(Exception):
    """No view contributed visibility above the floor; use the memory embedding."""

    def __init__(self, visibility_sum: float):
        self.visibility_sum = float(visibility_sum)
        super().__init__(f"total visibility {visibility_sum:.3g} at or below floor; "
                         "caller should fall back to the query's memory embedding")


# When the reference package is importable, raise ITS classes, so callers'
# ``except mvtrack3d.errors.NonFiniteWeight`` clauses catch the drop-in's
# errors too (the classes above are the same taxonomy, errors.py:10-46).
try:  # pragma: no cover - depends on the environment
    from mvtrack3d import errors as _ref_errors
except Exception:  # the reference is not installed: keep the local classes
    _ref_errors = None
if _ref_errors is not None:
    BehindCamera = _ref_errors.BehindCamera  # noqa: F811
    OffsetOutOfRange = _ref_errors.OffsetOutOfRange  # noqa: F811
    NonFiniteWeight = _ref_errors.NonFiniteWeight  # noqa: F811
    OddChannelCount = _ref_errors.OddChannelCount  # noqa: F811
    ChannelMismatch = _ref_errors.ChannelMismatch  # noqa: F811
    AllOccluded = _ref_errors.AllOccluded  # noqa: F811


class MsdaCudaError(RuntimeError):
    """The CUDA runtime reported a failure inside the C-ABI library."""


_BY_CODE = {
    L.MSDA_ODD_CHANNELS: OddChannelCount,
    L.MSDA_NONFINITE: NonFiniteWeight,
    L.MSDA_BAD_TARGET: ValueError,
    L.MSDA_ZERO_WEIGHT_SUM: ValueError,
    L.MSDA_BAD_PRECISION: ValueError,
    L.MSDA_CHANNEL_MISMATCH: ChannelMismatch,
    L.MSDA_CUDA_ERROR: MsdaCudaError,
    L.MSDA_BAD_ARG: ValueError,
    L.MSDA_OFFSET_RANGE: OffsetOutOfRange,
}


def raise_for_status(code: int, detail: int = -1, what: str = "") -> None:
    """Raise the reference exception class that matches a C-ABI status."""
    if code == L.MSDA_OK:
        return
    exc = _BY_CODE.get(int(code), RuntimeError)
    msg = L.status_string(code)
    if detail is not None and detail >= 0:
        unit = "query" if code in (L.MSDA_ZERO_WEIGHT_SUM, L.MSDA_BAD_ARG) else "sample"
        msg = f"{unit} {detail}: {msg}"
    if what:
        msg = f"{what}: {msg}"
    raise exc(msg)
