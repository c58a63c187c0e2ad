"""pytest plugin: run the REFERENCE's own test-suite with its hot path swapped
for this repo's GPU drop-in.

Loaded with ``-p dropin_pytest_plugin`` before collection, it rebinds
``mvtrack3d.features.msda_optimized`` / ``bilinear_sample`` (and, with
``DROPIN_ALL=1``, ``msda_reference``) — plus the names ``mvtrack3d.bench`` and
``mvtrack3d.oae`` imported from ``.features`` at import time — to
``paper_2601_10819_b200.features``.  The reference's objects
(``FeaturePyramid``, ``SamplePlan``, ``PrecisionMode``) go straight into the
drop-in, so the tests exercise exactly the call a reference maintainer would
redirect.  The reference package comes from ``baseline/_ref``
(the pip install of /root/reference); its tests from ``baseline/_ref_tests``
(a git-ignored copy, tools/run_reference_tests.py).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))

import mvtrack3d.bench as _rb  # noqa: E402
import mvtrack3d.features as _rf  # noqa: E402
import mvtrack3d.oae as _ro  # noqa: E402

from paper_2601_10819_b200 import features as _ours  # noqa: E402

SWAPPED = ["msda_optimized", "bilinear_sample"] + (["msda_reference"] if os.environ.get("DROPIN_ALL") == "1" else [])
for _name in SWAPPED:
    _fn = getattr(_ours, _name)
    for _mod in (_rf, _rb, _ro):
        if hasattr(_mod, _name):
            setattr(_mod, _name, _fn)


def pytest_report_header(config):
    return [f"dropin: mvtrack3d.features.{{{', '.join(SWAPPED)}}} -> paper_2601_10819_b200.features (GPU C ABI)"]
