"""GPU tests of the reference-facing drop-in (paper_2601_10819_b200.features)
beyond the MSDA calls: ``bilinear_sample`` bit for bit against the reference's
own outputs, the reference's error wording (first offending query named), and
malformed CSR plans rejected without touching memory outside the plan.
"""

import math

import numpy as np
import pytest

import helpers
from oracle import msda_oracle as mo

pytestmark = pytest.mark.gpu


def test_bilinear_sample_matches_reference_golden(golden, cuda_dev):
    """features.bilinear_sample on the GPU (C ABI msda_bilinear_host) returns
    the reference's bytes (features.py:184-219), signed zeros included, at
    random, integer, edge and out-of-grid coordinates."""
    from paper_2601_10819_b200 import features as F

    g = golden("bilinear")
    grids, coords = helpers.bilinear_inputs(np.random.default_rng(71))
    for k, (grid, (us, vs)) in enumerate(zip(grids, coords)):
        pyr = F.FeaturePyramid(0, [F.FeatureGrid(stride=4.0, values=grid)])
        got = np.stack([F.bilinear_sample(pyr, 0, float(u), float(v)) for u, v in zip(us, vs)])
        assert got.dtype == np.float32 and got.shape == g[f"out{k}"].shape
        assert got.tobytes() == g[f"out{k}"].tobytes(), k
    with pytest.raises(ValueError, match="finite"):
        F.bilinear_sample(pyr, 0, math.nan, 0.0)


def test_bilinear_sample_reads_page_locked_grids_in_place(cuda_dev):
    """A grid passed again is page-locked (features._HostPins) and then read
    in place by the kernel: same bytes, only the coordinates cross PCIe."""
    from paper_2601_10819_b200 import features as F

    rng = np.random.default_rng(72)
    grid = rng.standard_normal((512, 1024, 4)).astype(np.float32)  # 8 MB: above the pinning threshold
    pyr = F.FeaturePyramid(0, [F.FeatureGrid(stride=4.0, values=grid)])
    table, tiles = grid.reshape(-1, 4), [(0, 512, 1024)]
    for u, v in [(3.25, 7.5), (1023.0, 511.0), (-0.5, 200.75), (500.5, 100.25)]:
        got = F.bilinear_sample(pyr, 0, u, v)
        assert got.tobytes() == mo.bilinear_f32(table, tiles[0], u, v).tobytes()
    assert F.last_h2d_bytes(0) == 8  # the second call on: page-locked grid, two floats moved


def test_zero_weight_sum_names_first_query(cuda_dev):
    """The reference raises for the first offending query in order
    (features.py:264-269 / 285-287): the GPU status keeps the smallest."""
    from paper_2601_10819_b200 import features as F

    rng = np.random.default_rng(6)
    grids, _ = helpers.make_pyramids(rng, n_cams=1, n_levels=1)
    pyrs = [F.FeaturePyramid(0, [F.FeatureGrid(stride=4.0, values=grids[(0, 0)])])]
    ok = [(0, 0, 1.0, 1.0, 0.5)]
    zero = [(0, 0, 1.0, 1.0, 0.0), (0, 0, 2.0, 1.0, 0.0)]
    for bad in ([3, 700, 5], [999], [0, 1]):
        per_query = [zero if q in bad else ok for q in range(1000)]
        for prec in (F.PrecisionMode.FULL, F.PrecisionMode.PACKED_HALF):
            with pytest.raises(ValueError) as ei:
                F.msda_optimized(pyrs, F.SamplePlan(per_query), precision=prec)
            assert str(ei.value) == f"query {min(bad)}: plan weights sum to zero, cannot renormalize"


def test_malformed_csr_offsets_rejected(cuda_dev):
    """Decreasing / out-of-range device offsets report MSDA_BAD_ARG (ValueError)
    from the plan kernel (exact) or the gather (fast) instead of indexing
    outside the plan; the host entry point checks them before any copy."""
    import torch

    from paper_2601_10819_b200 import features as F
    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(8)
    grids, _ = helpers.make_pyramids(rng, n_cams=1, n_levels=1, channels=64)
    g = grids[(0, 0)]
    h, w, c = g.shape
    feats = ops.DeviceFeatures(torch.from_numpy(g.reshape(h * w, c)).to(cuda_dev),
                               torch.tensor([[[h, w]]], dtype=torch.int32), torch.zeros((1, 1), dtype=torch.int64))
    n = 6
    t = lambda a: torch.from_numpy(np.asarray(a)).to(cuda_dev)  # noqa: E731
    cols = [t(np.zeros(n, np.int32)), t(np.zeros(n, np.int32)), t(np.full(n, 1.5, np.float32)),
            t(np.full(n, 1.5, np.float32)), t(np.full(n, 0.5, np.float32))]
    for offs in ([0, 4, 2, 6], [0, 3, 9, 6], [-2, 3, 4, 6]):
        for prec in ("exact", "fast"):
            with pytest.raises(ValueError, match="invalid argument"):
                ops.msda_csr(feats, t(np.array(offs, np.int64)), *cols, precision=prec)
    out, empty = ops.msda_csr(feats, t(np.array([0, 2, 2, 6], np.int64)), *cols)  # the well-formed plan still runs
    assert empty.cpu().tolist() == [0, 1, 0]
    # host arrays: SamplePlan.from_csr validates the invariant
    with pytest.raises(ValueError, match="non-decreasing"):
        F.SamplePlan.from_csr([0, 4, 2], [0] * 4, [0] * 4, [1.0] * 4, [1.0] * 4, [1.0] * 4)


def test_oae_many_keypoints_single_level(cuda_dev):
    """L = 1 with more than 32 keypoints: the warp kernel's
    one-keypoint-per-lane projection cannot hold them, so the call takes the
    general kernel and matches the oracle (oae.py:81-164)."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(91)
    cams, channels = 3, 256
    grids = {(c, 0): rng.uniform(-1, 1, (64, 176, channels)).astype(np.float32) for c in range(cams)}
    shape = np.array([[[64, 176]]] * cams, dtype=np.int32)
    table, tiles = mo.pack_grids(grids, cams, 1)
    start = np.array([t[0] for t in tiles], dtype=np.int64).reshape(cams, 1)
    feats = ops.DeviceFeatures(torch.from_numpy(table).to(cuda_dev), torch.from_numpy(shape),
                               torch.from_numpy(start))
    from test_gpu_dense import _ring

    K, R, T = _ring(cams)
    camd = ops.Cameras(K, R, T, device=cuda_dev)
    q_n, n_learned = 5, 40  # P = 47 > 32
    anchors = np.zeros((q_n, 10), dtype=np.float32)
    anchors[:, 0:2] = rng.uniform(-3, 3, (q_n, 2))
    anchors[:, 2] = 0.9
    anchors[:, 3:6] = (0.6, 0.6, 1.8)
    anchors[:, 6] = rng.uniform(-math.pi, math.pi, q_n)
    offsets = rng.uniform(-1, 1, (n_learned, 3)).astype(np.float32)
    desc = rng.standard_normal((q_n, channels)).astype(np.float32)
    vis = rng.uniform(0.2, 1.0, (q_n, cams)).astype(np.float32)
    mem = rng.standard_normal((q_n, channels)).astype(np.float32)
    mem /= np.linalg.norm(mem, axis=1, keepdims=True)
    tt = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    emb, occl = ops.oae_pool(feats, tt(anchors), offsets, camd, [4.0], tt(desc), tt(vis), tt(mem))
    emb = emb.cpu().numpy()
    for q in range(q_n):
        kps = mo.keypoints(anchors[q].astype(np.float64), offsets.astype(np.float64))
        assert len(kps) == 7 + n_learned
        views = [mo.extract_view(table, tiles, 1, c, [4.0], K[c], R[c], T[c], kps, desc[q].astype(np.float64))
                 for c in range(cams)]
        ref, _ = mo.fuse(views, vis[q], mem[q])
        assert np.abs(emb[q] - ref).max() <= 1e-4, q


def test_partial_rejects_batch_mismatch(cuda_dev):
    """deformable_aggregation_partial checks the sampling batch against the
    feature table's (the C ABI takes the batch from the table descriptor)."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(12)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=1, n_q=4, n_p=3, cams=2, n_levels=2, groups=2, channels=8)
    table, tiles = mo.pack_grids(grids, 2, 2)
    start = np.array([t[0] for t in tiles], dtype=np.int64).reshape(2, 2)
    feats = ops.DeviceFeatures(torch.from_numpy(np.stack([table, table])).to(cuda_dev), torch.from_numpy(shape),
                               torch.from_numpy(start))
    with pytest.raises(ValueError, match="batch"):
        ops.deformable_aggregation_partial(feats, torch.from_numpy(loc).to(cuda_dev),
                                           torch.from_numpy(wts).to(cuda_dev))
