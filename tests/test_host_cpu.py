"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the host-side mirror of the reference API validates like the reference, and
the product never imports the oracle."""

import ast
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols():
    hdr = (ROOT / "include" / "msda_b200.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(msda_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_2601_10819_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = _declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table must mirror the header"


def test_status_strings_and_abi_version():
    from paper_2601_10819_b200 import _lib

    assert _lib.lib().msda_abi_version() == 2
    assert "zero" in _lib.status_string(_lib.MSDA_ZERO_WEIGHT_SUM)
    assert _lib.status_string(_lib.MSDA_OK) == "ok"


def test_argument_errors_without_gpu():
    """Host-side validation returns before touching the device."""
    from paper_2601_10819_b200 import _lib

    lib = _lib.lib()
    f = _lib.Features()
    p = _lib.CsrPlan()
    assert lib.msda_csr(ctypes.byref(f), ctypes.byref(p), 0, 1, None, None, None, 0, None) == _lib.MSDA_BAD_ARG
    f.data = 1
    f.spatial_shape = 1
    f.scale_start_index = 1
    f.n_cams = f.n_levels = f.batch = 1
    f.channels = 3
    f.n_rows = 4
    assert lib.msda_csr(ctypes.byref(f), ctypes.byref(p), 0, 1, None, None, None, 0, None) == _lib.MSDA_ODD_CHANNELS
    f.channels = 4
    assert lib.msda_csr(ctypes.byref(f), ctypes.byref(p), 7, 1, None, None, None, 0, None) == _lib.MSDA_BAD_PRECISION


def test_reference_mirror_validation():
    from paper_2601_10819_b200 import features as F
    from paper_2601_10819_b200.errors import NonFiniteWeight, OddChannelCount

    with pytest.raises(OddChannelCount):
        F.FeaturePyramid(0, [F.FeatureGrid(stride=8.0, values=np.zeros((2, 2, 3), np.float32))])
    g = F.FeatureGrid(stride=8.0, values=np.zeros((2, 2, 2), np.float32))
    with pytest.raises(ValueError):
        F.FeaturePyramid(0, [g, g])
    with pytest.raises(ValueError):
        F.FeatureGrid(stride=0.0, values=np.zeros((2, 2, 2), np.float32))
    with pytest.raises(NonFiniteWeight):
        F.SamplePlan([[(0, 0, 1.0, 1.0, np.nan)]])
    with pytest.raises(NonFiniteWeight):
        F.SamplePlan([[(0, 0, np.inf, 1.0, 1.0)]])
    assert F.pixel_to_cell(4.0, 8.0) == 0.0 and F.cell_to_pixel(0.0, 8.0) == 4.0
    per_query = [[(0, 0, 1.0, 2.0, 0.5), (1, 1, 0.5, 0.5, 0.25)], [], [(0, 1, 3.0, 0.0, 1.0)]]
    a = F.SamplePlan(per_query)
    flat = [(q, s) for q, ss in enumerate(per_query) for s in ss]
    b = F.SamplePlan.from_arrays([q for q, _ in flat][::-1], [s[0] for _, s in flat][::-1],
                                 [s[1] for _, s in flat][::-1], [s[2] for _, s in flat][::-1],
                                 [s[3] for _, s in flat][::-1], [s[4] for _, s in flat][::-1], 3)
    np.testing.assert_array_equal(a.offsets, b.offsets)
    assert a.num_samples == 3 and list(a.query_indices()) == [0, 0, 2]


def test_plan_target_errors_follow_reference_order():
    """features.py:229-236: sorted unique camera ids, first unknown id or first
    camera with an out-of-range level wins.  Host side only (no GPU call)."""
    from paper_2601_10819_b200 import features as F

    def pyr(cid, n_levels):
        return F.FeaturePyramid(cid, [F.FeatureGrid(stride=8.0 * 2**m, values=np.zeros((2, 2, 2), np.float32))
                                      for m in range(n_levels)])

    def err(pyrs, per_query):
        with pytest.raises(ValueError) as e:
            F._prepare(F._pyramid_map(pyrs), F.SamplePlan(per_query))
        return str(e.value)

    dense = [pyr(0, 2), pyr(1, 2)]
    assert err(dense, [[(7, 0, 1, 1, 1)], [(-1, 0, 1, 1, 1)]]) == "plan references unknown camera id -1"
    assert err(dense, [[(1, 2, 1, 1, 1)], [(5, 0, 1, 1, 1)]]) == "plan references a missing level of camera 1"
    assert err(dense, [[(5, 0, 1, 1, 1)], [(1, -1, 1, 1, 1)]]) == "plan references a missing level of camera 1"
    sparse = [pyr(3, 1), pyr(9, 3)]
    assert err(sparse, [[(9, 2, 1, 1, 1), (3, 1, 1, 1, 1)]]) == "plan references a missing level of camera 3"
    assert err(sparse, [[(9, 3, 1, 1, 1), (4, 0, 1, 1, 1)]]) == "plan references unknown camera id 4"
    ragged = [pyr(0, 1), pyr(1, 3)]
    assert err(ragged, [[(1, 2, 1, 1, 1), (0, 1, 1, 1, 1)]]) == "plan references a missing level of camera 0"
    F._prepare(F._pyramid_map(ragged), F.SamplePlan([[(1, 2, 1, 1, 1), (0, 0, 1, 1, 1)]]))
    # deferred: dense ids at full depth leave the range check to the device status
    F._prepare(F._pyramid_map(dense), F.SamplePlan([[(7, 0, 1, 1, 1)]]), defer_range_check=True)
    assert err(ragged, [[(0, 1, 1, 1, 1)]]) == "plan references a missing level of camera 0"


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2601_10819_b200"
    for py in pkg.rglob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            assert not any(n.split(".")[0] == "oracle" for n in names), f"{py} imports the oracle"


def test_bench_reference_arm_contract():
    """bench.py --impl reference runs on the host alone (the reference's CPU
    algorithm): one JSON line with the contract's keys, impl "reference",
    an e2e object with zero transfer bytes and a cpu_baseline describing it."""
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "default",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "default"
    # the real reference (baseline/_ref) is timed when installed, else the oracle port
    assert d["cpu_baseline"]["kind"] == ("reference" if (ROOT / "baseline" / "_ref" / "mvtrack3d").exists()
                                         else "port")
    assert "cpu_model" in d["cpu_baseline"]["host"] or d["cpu_baseline"]["host"]["cpu_count"] >= 1


def test_bench_launches_n_ranks():
    """bench.py --gpus 2 without torchrun re-launches itself with 2 ranks
    (torch.distributed.run, 127.0.0.1): the gloo plumbing mode prints one
    JSON line with n_gpus = 2; without GPUs and without the fold flag the
    launcher refuses loudly instead of timing one rank."""
    import json
    import os
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env={**env, "BENCH_PLUMBING": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] is None and "no measurement" in d["data"]
    import torch

    if torch.cuda.device_count() < 2:
        r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                           capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
        assert r.returncode == 2 and "one rank per GPU" in r.stderr


def test_sample_plan_from_csr_validates_offsets():
    """SamplePlan.from_csr enforces the CSR invariant the reference's
    constructors establish (features.py:122-171): offsets start at 0, never
    decrease, and end at the per-sample array length."""
    from paper_2601_10819_b200 import features as F

    one = [1.0] * 3
    F.SamplePlan.from_csr([0, 1, 3], [0] * 3, [0] * 3, one, one, one)
    for offs in ([1, 2, 3], [0, 2, 1, 3], [0, 1, 4]):
        with pytest.raises(ValueError):
            F.SamplePlan.from_csr(offs, [0] * 3, [0] * 3, one, one, one)
    with pytest.raises(ValueError):
        F.SamplePlan.from_csr([0, 3], [0] * 3, [0] * 3, one, one, [1.0, 1.0])


def test_bilinear_oracle_matches_reference_golden(golden):
    """The numpy restatement of bilinear_sample equals the reference's bytes."""
    import sys

    sys.path.insert(0, str(ROOT / "tests"))
    import helpers
    from oracle import msda_oracle as mo

    g = golden("bilinear")
    grids, coords = helpers.bilinear_inputs(np.random.default_rng(71))
    for k, (grid, (us, vs)) in enumerate(zip(grids, coords)):
        h, w, c = grid.shape
        got = np.stack([mo.bilinear_f32(grid.reshape(h * w, c), (0, h, w), u, v) for u, v in zip(us, vs)])
        assert got.tobytes() == g[f"out{k}"].tobytes(), k
