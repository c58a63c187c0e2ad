"""GPU checks of the properties the reference pins in pkg/tests/test_features.py
(bilinear identities, zero padding, convexity, scaling) plus edge cases of the
exact kernels (huge coordinates, non-finite features, batch offsets, the
device API in PACKED_HALF mode)."""

import numpy as np
import pytest

import helpers
from oracle import msda_oracle as mo

pytestmark = pytest.mark.gpu


def _pyr(F, vals, stride=8.0):
    return [F.FeaturePyramid(0, [F.FeatureGrid(stride=stride, values=vals)])]


def test_bilinear_identities(cuda_dev):
    """test_features.py:66-95: cell centres, 4-cell midpoint, far outside,
    half mass past the last column — through the exact GPU path."""
    from paper_2601_10819_b200 import features as F

    rng = np.random.default_rng(0)
    vals = rng.standard_normal((4, 5, 6)).astype(np.float32)
    per_query = [[(0, 0, float(u), float(v), 1.0)] for v in range(4) for u in range(5)]
    out, _ = F.msda_optimized(_pyr(F, vals), F.SamplePlan(per_query))
    np.testing.assert_array_equal(out, vals.reshape(20, 6))
    mid, _ = F.msda_optimized(_pyr(F, vals), F.SamplePlan([[(0, 0, 0.5, 0.5, 1.0)]]))
    np.testing.assert_allclose(mid[0], (vals[0, 0] + vals[0, 1] + vals[1, 0] + vals[1, 1]) / 4.0, rtol=1e-6)
    ones = np.ones((3, 3, 2), dtype=np.float32)
    far, _ = F.msda_optimized(_pyr(F, ones), F.SamplePlan([[(0, 0, -5.0, -5.0, 1.0)], [(0, 0, 10.0, 1.0, 1.0)]]))
    np.testing.assert_array_equal(far, 0.0)
    edge, _ = F.msda_optimized(_pyr(F, ones), F.SamplePlan([[(0, 0, 2.5, 1.0, 1.0)]]))
    np.testing.assert_allclose(edge[0], [0.5, 0.5], rtol=1e-6)


def test_convexity_and_unnormalized_scaling(cuda_dev):
    """test_features.py:273-313."""
    from paper_2601_10819_b200 import features as F

    rng = np.random.default_rng(12)
    for _ in range(10):
        vals = rng.standard_normal((int(rng.integers(4, 7)), int(rng.integers(4, 7)), 4)).astype(np.float32)
        h, w, _ = vals.shape
        samples = [(0, 0, float(rng.uniform(0, w - 1)), float(rng.uniform(0, h - 1)), float(rng.uniform(0.1, 1)))
                   for _ in range(6)]
        out, _ = F.msda_optimized(_pyr(F, vals), F.SamplePlan([samples]))
        flat = vals.reshape(-1, 4)
        assert np.all(out[0] >= flat.min(axis=0) - 1e-6) and np.all(out[0] <= flat.max(axis=0) + 1e-6)
    samples = [(0, 0, 1.0, 1.0, 0.25), (0, 0, 0.5, 0.5, 0.5)]
    o1, _ = F.msda_optimized(_pyr(F, vals), F.SamplePlan([samples]), normalize=False)
    o2, _ = F.msda_optimized(_pyr(F, vals), F.SamplePlan([[(c, m, u, v, 2 * w_) for c, m, u, v, w_ in samples]]),
                             normalize=False)
    np.testing.assert_allclose(o2, 2.0 * o1, rtol=1e-6)


def test_huge_and_negative_coordinates_and_weights(c_oracle, cuda_dev):
    """Coordinates far beyond int range must not overflow (features.py:318-321);
    negative weights and negative weight sums follow the reference bit for bit."""
    from paper_2601_10819_b200 import features as F

    rng = np.random.default_rng(3)
    vals = rng.standard_normal((6, 7, 8)).astype(np.float32)
    per_query = [
        [(0, 0, 3e30, 1.0, 1.0), (0, 0, -3e30, -2e9, 0.5), (0, 0, 2.0, 3.0, 0.25)],
        [(0, 0, 1.5, 2.5, -0.75), (0, 0, 0.25, 4.5, 0.5)],            # negative weight, positive sum
        [(0, 0, 1.5, 2.5, -0.75), (0, 0, 0.25, 4.5, -0.5)],           # negative sum
        [(0, 0, 6.0, 5.0, 1.0), (0, 0, -1.0, -1.0, 1.0), (0, 0, 5.999999, 4.5, 1.0)],
    ]
    plan = F.SamplePlan(per_query)
    out, _ = F.msda_optimized(_pyr(F, vals), plan)
    table, tiles = mo.pack_grids({(0, 0): vals}, 1, 1)
    ref, _ = c_oracle.msda_c(table, tiles, 1, plan.offsets, plan.camera_ids, plan.levels, plan.us, plan.vs,
                             plan.weights)
    assert out.tobytes() == ref.tobytes()


def test_nonfinite_features_propagate_like_the_reference(cuda_dev):
    """0 * inf = nan for an in-grid corner with zero interpolation weight;
    out-of-grid corners read exact zeros (features.py:214-219)."""
    from paper_2601_10819_b200 import features as F

    vals = np.ones((3, 3, 2), dtype=np.float32)
    vals[1, 2] = np.inf
    out, _ = F.msda_optimized(_pyr(F, vals), F.SamplePlan([[(0, 0, 1.0, 1.0, 1.0)], [(0, 0, 0.0, 0.0, 1.0)]]))
    assert np.isnan(out[0]).all()  # corner (x=2, y=1) is in the grid with weight 0: 0 * inf
    np.testing.assert_array_equal(out[1], 1.0)


def test_device_api_packed_half_and_batches(golden, c_oracle, cuda_dev):
    """ops.msda_csr in EXACT_HALF on f16 tables equals the reference PACKED_HALF
    bytes; CSR queries address per-batch tables through queries_per_batch."""
    import torch

    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.workload import BenchWorkload, generate_workload

    g = golden("bench")
    wl = BenchWorkload(cameras=3, levels=4, channels=32, queries=40, points_per_query=13, level0_size=(32, 88))
    gw = generate_workload(wl)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda_dev)  # noqa: E731
    feats = ops.DeviceFeatures(t(gw.table).half(), t(gw.spatial_shape), t(gw.tile_start.reshape(3, 4)))
    out, _ = ops.msda_csr(feats, t(gw.offsets), t(gw.camera_ids), t(gw.levels), t(gw.us), t(gw.vs), t(gw.weights),
                          precision="exact_half")
    assert out.cpu().numpy().tobytes() == g["medium_half"].tobytes()


def test_exact_dense_batches_use_their_own_tables(cuda_dev):
    """Batch b's queries must read batch b's table (row_base offsets)."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(9)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=3, n_q=5, n_p=4, cams=2, n_levels=2, groups=2, channels=8)
    table, tiles = mo.pack_grids(grids, 2, 2)
    tables = np.stack([table * np.float32(b + 1) for b in range(3)])  # distinct per batch (exact scaling)
    start = np.array([t_[0] for t_ in tiles], dtype=np.int64).reshape(2, 2)
    feats = ops.DeviceFeatures(torch.from_numpy(tables).to(cuda_dev), torch.from_numpy(shape),
                               torch.from_numpy(start))
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    for prec in ("exact", "fast"):
        out = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision=prec,
                                         check=True).cpu().numpy()
        for b in range(3):
            ref = mo.msda_dense_groups(tables[b], tiles, shape, loc[b:b + 1], wts[b:b + 1], 2)[0]
            if prec == "exact":
                assert out[b].tobytes() == ref.tobytes()
            else:
                assert np.abs(out[b] - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max())
