#!/usr/bin/env python
"""Run the reference's own tests against the GPU drop-in.

    python tools/run_reference_tests.py --stage      # here: copy /root/reference/pkg/tests -> baseline/_ref_tests
    python tools/run_reference_tests.py [pytest args] # on the GPU box

``baseline/_ref`` holds the pip install of the reference and
``baseline/_ref_tests`` a git-ignored copy of its tests; both travel to the
GPU box with the gpurun snapshot.  The tests run under
``tools/dropin_pytest_plugin.py``, which swaps ``msda_optimized`` and
``bilinear_sample`` (``DROPIN_ALL=1``: ``msda_reference`` too) for the drop-in.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
TESTS = ROOT / "baseline" / "_ref_tests"
# the hot-path tests: features, bench, OAE, and acceptance criteria 1-3
DEFAULT = ["test_features.py", "test_bench.py", "test_oae.py",
           "test_acceptance.py::test_criterion_1_msda_parity", "test_acceptance.py::test_criterion_2_msda_throughput",
           "test_acceptance.py::test_criterion_3_visibility_and_fusion"]


def main():
    if sys.argv[1:2] == ["--stage"]:
        src = Path(os.environ.get("MVTRACK3D_TESTS", "/root/reference/pkg/tests"))
        if TESTS.exists():
            shutil.rmtree(TESTS)
        shutil.copytree(src, TESTS, ignore=shutil.ignore_patterns("__pycache__"))
        print(f"staged {src} -> {TESTS}")
        return 0
    if not (ROOT / "baseline" / "_ref" / "mvtrack3d").exists() or not TESTS.exists():
        print("baseline/_ref or baseline/_ref_tests missing: install the reference and run --stage first",
              file=sys.stderr)
        return 2
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tools"), str(ROOT / "baseline" / "_ref"), str(ROOT),
                                         str(TESTS), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    args = sys.argv[1:] or DEFAULT
    cmd = [sys.executable, "-m", "pytest", "-p", "dropin_pytest_plugin", "-p", "no:cacheprovider", "-q",
           "--rootdir", str(TESTS), *[a if a.startswith("-") else str(TESTS / a) for a in args]]
    return subprocess.call(cmd, env=env, cwd=str(TESTS))


if __name__ == "__main__":
    sys.exit(main())
