"""GPU parity of the Sparse4D dense path (deformable_aggregation), the fused
projection path and OAE pooling.

Oracles: the reference itself (tests/golden/dense.npz, oae.npz) and the
numpy oracle (oracle/msda_oracle.py) composed as SURVEY §8(c) prescribes.
Bars: EXACT bitwise; FAST fp32 1e-4 relative (max|d| / max|ref|); f16/bf16
storage 1e-2 (max|d| / max(1, max|ref|)); projection / OAE (f64 in the
reference) 1e-4 relative.
"""

import math

import numpy as np
import pytest

import helpers
from oracle import msda_oracle as mo

pytestmark = pytest.mark.gpu


def _feats(ops, torch, grids, shape, dev, dtype=None, batch=1):
    import torch as _t

    cams, n_levels = shape.shape[:2]
    table, tiles = mo.pack_grids(grids, cams, n_levels)
    start = np.array([t[0] for t in tiles], dtype=np.int64).reshape(cams, n_levels)
    tt = _t.from_numpy(np.ascontiguousarray(np.broadcast_to(table, (batch,) + table.shape))).to(dev)
    if dtype is not None:
        tt = tt.to(dtype)
    return ops.DeviceFeatures(tt.contiguous(), _t.from_numpy(shape), _t.from_numpy(start)), table, tiles


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


def test_dense_exact_matches_reference_golden(golden, cuda_dev):
    import torch

    from paper_2601_10819_b200 import ops

    g = golden("dense")["out"]
    rng = np.random.default_rng(31)
    pos = 0
    for i in range(6):
        groups = (1, 2, 4)[i % 3]
        bs = 1 + i % 2
        grids, shape, loc, wts = helpers.make_dense(rng, bs=bs, n_q=4, n_p=3, cams=2, n_levels=2, groups=groups,
                                                    channels=8)
        feats, _, _ = _feats(ops, torch, grids, shape, cuda_dev, batch=bs)
        for normalize in (False, True):
            out = ops.deformable_aggregation(feats, None, None, torch.from_numpy(loc).to(cuda_dev),
                                             torch.from_numpy(wts).to(cuda_dev), precision="exact",
                                             normalize=normalize, check=True).cpu().numpy().reshape(-1)
            assert out.tobytes() == g[pos:pos + out.size].tobytes(), (i, normalize)
            pos += out.size


@pytest.mark.parametrize("groups,channels,cams,levels,normalize", [
    (8, 256, 6, 4, False), (8, 256, 3, 4, True), (1, 64, 2, 3, False), (4, 32, 4, 2, True), (2, 8, 2, 2, False),
    (16, 256, 3, 4, True), (2, 128, 2, 4, True)])
def test_dense_fast_fp32_tolerance(cuda_dev, groups, channels, cams, levels, normalize):
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(100 + groups + channels)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=2, n_q=7, n_p=13, cams=cams, n_levels=levels, groups=groups,
                                                channels=channels, size_lo=6, size_hi=30)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, batch=2)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    fast = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision="fast", normalize=normalize,
                                      check=True).cpu().numpy()
    exact = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision="exact", normalize=normalize,
                                       check=True).cpu().numpy()
    ref = mo.msda_dense_groups(table, tiles, shape, loc, wts, levels, normalize=normalize)
    assert exact.tobytes() == ref.tobytes()
    assert rel(fast, ref) <= 1e-4


@pytest.mark.parametrize("dt", ["float16", "bfloat16"])
def test_dense_fast_half_storage(cuda_dev, dt):
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(7)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=1, n_q=16, n_p=13, cams=6, n_levels=4, groups=8,
                                                channels=256, size_lo=8, size_hi=40)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, dtype=getattr(torch, dt))
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    out = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), check=True).cpu().numpy()
    ref = mo.msda_dense_groups(table, tiles, shape, loc, wts, 4)
    assert np.abs(out - ref).max() / max(1.0, np.abs(ref).max()) <= 1e-2
    rounded = feats.table[0].float().cpu().numpy()
    ref_r = mo.msda_dense_groups(rounded, tiles, shape, loc, wts, 4)
    assert rel(out, ref_r) <= 1e-4  # only summation order / FMA differ from the pre-rounded reference
    ex = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision="exact", check=True).cpu().numpy()
    assert ex.tobytes() == ref_r.tobytes()
    # the paper's half2 accumulation (f16 products and per-camera partials): north_star fp16 bound only
    h2 = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision="fast_h2", check=True).cpu().numpy()
    assert np.abs(h2 - ref).max() / max(1.0, np.abs(ref).max()) <= 1e-2


def _ring(n, radius=12.0, height=4.0, focal=300.0, size=(704, 256)):
    """camera_looking_at ring (geometry.py:258-290) restated for the test."""
    Ks, Rs, ts = [], [], []
    for i in range(n):
        ang = 2 * math.pi * i / n
        pos = np.array([radius * math.cos(ang), radius * math.sin(ang), height])
        fwd = np.array([0.0, 0.0, 0.9]) - pos
        z = fwd / np.linalg.norm(fwd)
        x = np.cross(z, [0.0, 0.0, 1.0])
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R = np.vstack([x, y, z])
        Ks.append([focal, focal, size[0] / 2, size[1] / 2])
        Rs.append(R)
        ts.append(-R @ pos)
    return np.array(Ks), np.array(Rs), np.array(ts)


@pytest.mark.parametrize("normalize,channels,groups", [(False, 64, 4), (True, 64, 4), (False, 256, 8),
                                                      (True, 256, 8)])
def test_dense_project_matches_composed_oracle(cuda_dev, normalize, channels, groups):
    """Fused keypoints + projection (msda_dense_project) against the composed
    oracle.  C = 256 takes the projection pre-pass + pipelined gather; C = 64
    the anchor-major fused kernel."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(55)
    cams, n_levels = 4, 4
    strides = [4.0, 8.0, 16.0, 32.0]
    grids = {}
    shape = np.zeros((cams, n_levels, 2), dtype=np.int32)
    for c in range(cams):
        for m, s in enumerate(strides):
            h, w = int(math.ceil(256 / s)), int(math.ceil(704 / s))
            grids[(c, m)] = rng.uniform(-1, 1, (h, w, channels)).astype(np.float32)
            shape[c, m] = (h, w)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev)
    K, R, T = _ring(cams)
    q_n = 24
    anchors = np.zeros((1, q_n, 10), dtype=np.float32)
    anchors[0, :, 0:2] = rng.uniform(-4, 4, (q_n, 2))
    anchors[0, :, 2] = 0.9
    anchors[0, :, 3:6] = (0.6, 0.6, 1.8)
    anchors[0, :, 6] = rng.uniform(-math.pi, math.pi, q_n)
    anchors[0, :, 7:9] = rng.uniform(-1, 1, (q_n, 2))
    anchors[0, 3, 0:3] = (12.0 * math.cos(0.0), 0.0, 4.5)  # near camera 0: partly behind it
    offsets = rng.uniform(-1, 1, (6, 3)).astype(np.float32)
    wts = rng.uniform(0.01, 1.0, (1, q_n, 13, cams, n_levels, groups)).astype(np.float32)
    camd = ops.Cameras(K, R, T, device=cuda_dev)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    ref = mo.msda_project_groups(table, tiles, anchors, offsets, K, R, T, strides, wts, n_levels, normalize, 0.1)
    for prec in ("fast", "exact"):
        out = ops.msda_dense_project(feats, t(anchors), offsets, camd, strides, t(wts), dt=0.1, precision=prec,
                                     normalize=normalize, check=True).cpu().numpy()
        assert rel(out, ref) <= 1e-4, prec


@pytest.mark.parametrize("channels", [256, 64])
def test_dense_project_offset_out_of_range(cuda_dev, channels):
    """A learned offset component beyond [-1, 1] raises the reference's
    OffsetOutOfRange (geometry.py:241-244) on every projected path (pre-pass +
    staged split at C = 256, the fused kernel at C = 64; FAST and EXACT), and
    the next valid call on the same workspace succeeds (its status reset)."""
    import torch

    from paper_2601_10819_b200 import errors, ops

    rng = np.random.default_rng(56)
    cams, n_levels, groups = 4, 4, 8
    grids, shape = {}, np.zeros((cams, n_levels, 2), dtype=np.int32)
    for c in range(cams):
        for m, s in enumerate([4.0, 8.0, 16.0, 32.0]):
            h, w = int(math.ceil(256 / s)), int(math.ceil(704 / s))
            grids[(c, m)] = rng.uniform(-1, 1, (h, w, channels)).astype(np.float32)
            shape[c, m] = (h, w)
    feats, _, _ = _feats(ops, torch, grids, shape, cuda_dev)
    K, R, T = _ring(cams)
    anchors = np.zeros((1, 8, 10), dtype=np.float32)
    anchors[0, :, 0:2] = rng.uniform(-4, 4, (8, 2))
    anchors[0, :, 2:6] = (0.9, 0.6, 0.6, 1.8)
    good = rng.uniform(-1, 1, (6, 3)).astype(np.float32)
    bad = good.copy()
    bad[4, 1] = 1.25
    wts = torch.from_numpy(rng.uniform(0.01, 1.0, (1, 8, 13, cams, n_levels, groups)).astype(np.float32)).to(cuda_dev)
    camd = ops.Cameras(K, R, T, device=cuda_dev)
    an = torch.from_numpy(anchors).to(cuda_dev)
    for prec in ("fast", "exact"):
        with pytest.raises(errors.OffsetOutOfRange):
            ops.msda_dense_project(feats, an, bad, camd, [4.0, 8.0, 16.0, 32.0], wts, precision=prec, check=True)
        out = ops.msda_dense_project(feats, an, good, camd, [4.0, 8.0, 16.0, 32.0], wts, precision=prec, check=True)
        assert torch.isfinite(out).all()


def test_oae_pool_matches_reference_golden(golden, cuda_dev):
    import torch

    from paper_2601_10819_b200 import ops

    g = golden("oae")
    n_cams, n_levels = len(g["K"]), len(g["strides"])
    grids, pos = {}, 0
    shape = np.zeros((n_cams, n_levels, 2), dtype=np.int32)
    for i, (h, w) in enumerate(g["shapes"]):
        n = h * w * 16
        grids[(i // n_levels, i % n_levels)] = g["grids"][pos:pos + n].reshape(h, w, 16).astype(np.float32)
        shape[i // n_levels, i % n_levels] = (h, w)
        pos += n
    feats, _, _ = _feats(ops, torch, grids, shape, cuda_dev)
    camd = ops.Cameras(g["K"], g["R"], g["t"], device=cuda_dev)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda_dev)  # noqa: E731
    emb, occl = ops.oae_pool(feats, t(g["anchors"].astype(np.float32)), g["offsets"].astype(np.float32), camd,
                             g["strides"].astype(np.float32), t(g["desc"].astype(np.float32)),
                             t(g["vis"].astype(np.float32)), t(g["memory"].astype(np.float32)))
    emb, occl = emb.cpu().numpy(), occl.cpu().numpy()
    assert list(occl) == [bool(x) for x in g["occluded"]]
    for q in range(len(emb)):
        if occl[q]:
            np.testing.assert_allclose(emb[q], g["memory"][q], rtol=1e-6, atol=1e-7)
        else:
            assert np.abs(emb[q] - g["emb"][q]).max() <= 1e-4  # unit vectors: absolute == relative


def test_oae_channel_mismatch(cuda_dev):
    import torch

    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.errors import ChannelMismatch

    rng = np.random.default_rng(3)
    grids = {(0, 0): rng.standard_normal((8, 8, 4)).astype(np.float32)}
    feats, _, _ = _feats(ops, torch, grids, np.array([[[8, 8]]], dtype=np.int32), cuda_dev)
    camd = ops.Cameras([[100, 100, 64, 64]], np.eye(3).reshape(1, 9), [[0, 0, 0]], device=cuda_dev)
    with pytest.raises(ChannelMismatch):
        ops.oae_pool(feats, torch.zeros(1, 10), np.zeros((0, 3)), camd, [8.0], torch.zeros(1, 6), torch.ones(1, 1),
                     torch.zeros(1, 4))


@pytest.mark.parametrize("dt,cams", [("float32", 10), ("bfloat16", 10), ("float32", 6), ("bfloat16", 17)])
def test_oae_pool_production_kernel(cuda_dev, dt, cams):
    """C = 256 takes the warp-per-camera online-softmax kernel (more than 8
    cameras: per-camera-group CTAs + the finishing reduction); compare with
    the oracle (oae.py:81-164 restated) on the features the GPU sees."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(61)
    n_levels, channels = 4, 256
    strides = [4.0, 8.0, 16.0, 32.0]
    grids, shape = {}, np.zeros((cams, n_levels, 2), dtype=np.int32)
    for c in range(cams):
        for m, s in enumerate(strides):
            h, w = int(math.ceil(256 / s)), int(math.ceil(704 / s))
            grids[(c, m)] = rng.uniform(-1, 1, (h, w, channels)).astype(np.float32)
            shape[c, m] = (h, w)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, dtype=getattr(torch, dt))
    seen = feats.table[0].float().cpu().numpy()
    K, R, T = _ring(cams)
    camd = ops.Cameras(K, R, T, device=cuda_dev)
    q_n = 12
    anchors = np.zeros((q_n, 10), dtype=np.float32)
    anchors[:, 0:2] = rng.uniform(-4, 4, (q_n, 2))
    anchors[:, 2] = 0.9
    anchors[:, 3:6] = (0.6, 0.6, 1.8)
    anchors[:, 6] = rng.uniform(-math.pi, math.pi, q_n)
    offsets = rng.uniform(-1, 1, (6, 3)).astype(np.float32)
    desc = rng.standard_normal((q_n, channels)).astype(np.float32)
    vis = rng.uniform(0.0, 1.0, (q_n, cams)).astype(np.float32)
    vis[4] = 1e-5  # all occluded -> memory
    mem = rng.standard_normal((q_n, channels)).astype(np.float32)
    mem /= np.linalg.norm(mem, axis=1, keepdims=True)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    emb, occl = ops.oae_pool(feats, t(anchors), offsets, camd, strides, t(desc), t(vis), t(mem))
    emb, occl = emb.cpu().numpy(), occl.cpu().numpy()
    for q in range(q_n):
        kps = mo.keypoints(anchors[q].astype(np.float64), offsets.astype(np.float64))
        views = [mo.extract_view(seen, tiles, n_levels, c, strides, K[c], R[c], T[c], kps, desc[q].astype(np.float64))
                 for c in range(cams)]
        ref, ref_occ = mo.fuse(views, vis[q], mem[q])
        assert bool(occl[q]) == ref_occ
        assert np.abs(emb[q] - ref).max() <= 1e-4, q


@pytest.mark.parametrize("cams", [6, 17])
def test_oae_pool_offset_out_of_range(cuda_dev, cams):
    """An out-of-range learned offset raises OffsetOutOfRange (geometry.py:241-
    244) from the warp kernel, single CTA per query (6 cameras) and split over
    camera groups (17, where the kernel's first thread resets the status);
    the next valid call on the same workspace succeeds."""
    import torch

    from paper_2601_10819_b200 import errors, ops

    rng = np.random.default_rng(62)
    n_levels, channels, strides = 4, 256, [4.0, 8.0, 16.0, 32.0]
    grids, shape = {}, np.zeros((cams, n_levels, 2), dtype=np.int32)
    for c in range(cams):
        for m, s in enumerate(strides):
            h, w = int(math.ceil(256 / s)), int(math.ceil(704 / s))
            grids[(c, m)] = rng.uniform(-1, 1, (h, w, channels)).astype(np.float32)
            shape[c, m] = (h, w)
    feats, _, _ = _feats(ops, torch, grids, shape, cuda_dev, dtype=torch.bfloat16)
    K, R, T = _ring(cams)
    camd = ops.Cameras(K, R, T, device=cuda_dev)
    q_n = 5
    anchors = np.zeros((q_n, 10), dtype=np.float32)
    anchors[:, 0:2] = rng.uniform(-4, 4, (q_n, 2))
    anchors[:, 2:6] = (0.9, 0.6, 0.6, 1.8)
    good = rng.uniform(-1, 1, (6, 3)).astype(np.float32)
    bad = good.copy()
    bad[2, 0] = -1.5
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    desc, vis = t(rng.standard_normal((q_n, channels)).astype(np.float32)), t(np.ones((q_n, cams), np.float32))
    mem = rng.standard_normal((q_n, channels)).astype(np.float32)
    mem = t(mem / np.linalg.norm(mem, axis=1, keepdims=True))
    with pytest.raises(errors.OffsetOutOfRange):
        ops.oae_pool(feats, t(anchors), bad, camd, strides, desc, vis, mem)
    emb, _ = ops.oae_pool(feats, t(anchors), good, camd, strides, desc, vis, mem)
    assert torch.isfinite(emb).all()


def _uniform_grids(rng, cams, levels, channels):
    grids = {}
    shape = np.zeros((cams, len(levels), 2), dtype=np.int32)
    for c in range(cams):
        for m, (h, w) in enumerate(levels):
            grids[(c, m)] = rng.uniform(-1, 1, (h, w, channels)).astype(np.float32)
            shape[c, m] = (h, w)
    return grids, shape


@pytest.mark.parametrize("dt,precision,normalize,channels,groups", [
    ("float32", "fast", False, 256, 8), ("float32", "fast", True, 256, 8), ("float32", "fast", False, 128, 4),
    ("float16", "fast", False, 256, 8), ("float16", "fast_h2", False, 256, 8), ("bfloat16", "fast", True, 256, 8)])
def test_dense_slice_kernel(cuda_dev, dt, precision, normalize, channels, groups):
    """Equal level shapes on every camera select the coarse-level staging
    kernel (camera x channel-slice CTAs, red.add partials)."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(71)
    cams, levels = 5, [(32, 88), (16, 44), (8, 22), (4, 11)]
    grids, shape = _uniform_grids(rng, cams, levels, channels)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, dtype=getattr(torch, dt), batch=2)
    seen = feats.table[0].float().cpu().numpy()
    bs, q_n, p_n = 2, 40, 13
    loc = rng.uniform(-0.05, 1.05, (bs, q_n, p_n, cams, 2)).astype(np.float32)
    logits = rng.standard_normal((bs, q_n, p_n * cams * 4, groups))
    e = np.exp(logits - logits.max(axis=2, keepdims=True))
    wts = (e / e.sum(axis=2, keepdims=True)).reshape(bs, q_n, p_n, cams, 4, groups).astype(np.float32)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    out = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision=precision, normalize=normalize,
                                     check=True).cpu().numpy()
    ref = mo.msda_dense_groups(seen, tiles, shape, loc, wts, 4, normalize=normalize)
    tol = 1e-2 if precision == "fast_h2" else 1e-4
    assert rel(out, ref) <= tol


@pytest.mark.parametrize("dt,groups,normalize", [("float32", 8, True), ("float32", 8, False), ("float32", 1, True),
                                                 ("float32", 4, True), ("float16", 8, True), ("bfloat16", 2, False)])
def test_dense_exact_one_pass_with_ties(cuda_dev, dt, groups, normalize):
    """EXACT with channel groups canonicalises once for every group: samples
    whose (camera, level, v, u) tie are ordered per group by that group's
    weight.  Duplicated sampling points (exact ties, with and without equal
    weights) must still give the per-group reference bytes."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(17 + groups)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=2, n_q=9, n_p=13, cams=3, n_levels=4, groups=groups,
                                                channels=256, size_lo=6, size_hi=20)
    loc[:, :, 5] = loc[:, :, 2]  # point 5 duplicates point 2 in every camera: (v, u) ties in every level
    loc[:, :, 9] = loc[:, :, 2]
    wts[:, :, 9] = wts[:, :, 2]  # ... one duplicate with the very same weights
    wts[0, 3, 5, :, :, 0] = wts[0, 3, 2, :, :, 0]  # equal weight in one group only
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, dtype=getattr(torch, dt), batch=2)
    seen = feats.table[0].float().cpu().numpy()
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    out = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision="exact", normalize=normalize,
                                     check=True).cpu().numpy()
    ref = mo.msda_dense_groups(seen, tiles, shape, loc, wts, 4, normalize=normalize)
    assert out.tobytes() == ref.tobytes()


def test_camera_sharded_partials_on_device(cuda_dev):
    """The camera-sharded driver's device path (single rank: no all-reduce):
    msda_dense_partial numerators + weight sums, then msda_dense_normalize —
    equals the normalised one-call aggregation; zero sums raise."""
    import torch

    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.dist import CameraShardedAggregation

    rng = np.random.default_rng(29)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=2, n_q=10, n_p=13, cams=4, n_levels=4, groups=8,
                                                channels=256, size_lo=6, size_hi=24)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, batch=2)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    part, wsum = ops.deformable_aggregation_partial(feats, t(loc), t(wts))
    assert np.allclose(wsum.cpu().numpy(), wts.sum(axis=(2, 3, 4)), rtol=1e-5)
    agg = CameraShardedAggregation.for_device_features(4, feats)
    out = agg(t(loc), t(wts), normalize=True).cpu().numpy()
    ref = mo.msda_dense_groups(table, tiles, shape, loc, wts, 4, normalize=True)
    assert rel(out, ref) <= 1e-4
    raw = agg(t(loc), t(wts), normalize=False).cpu().numpy()
    assert rel(raw, mo.msda_dense_groups(table, tiles, shape, loc, wts, 4, normalize=False)) <= 1e-4
    zero = wts.copy()
    zero[1, 3, :, :, :, 2] = 0.0
    with pytest.raises(ValueError, match="sum to zero"):
        agg(t(loc), t(zero), normalize=True)


@pytest.mark.parametrize("dt", ["float32", "float16"])
def test_dense_exact_full_size_cfg1(c_oracle, cuda_dev, dt):
    """BASELINE configs[0] at full size (6 cams, 64x176 .. 8x22, 900 anchors,
    13 points, C = 256, G = 8), EXACT, normalised: GPU bytes == per-group C
    oracle bytes on the features the GPU sees."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(2601)
    cams, levels, C, G, Q, P = 6, [(64, 176), (32, 88), (16, 44), (8, 22)], 256, 8, 900, 13
    grids, shape = _uniform_grids(rng, cams, levels, C)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, dtype=getattr(torch, dt))
    seen = feats.table[0].float().cpu().numpy()
    loc = rng.uniform(-0.02, 1.02, (1, Q, P, cams, 2)).astype(np.float32)
    logits = rng.standard_normal((1, Q, P * cams * 4, G))
    e = np.exp(logits - logits.max(axis=2, keepdims=True))
    wts = (e / e.sum(axis=2, keepdims=True)).reshape(1, Q, P, cams, 4, G).astype(np.float32)
    out = ops.deformable_aggregation(feats, None, None, torch.from_numpy(loc).to(cuda_dev),
                                     torch.from_numpy(wts).to(cuda_dev), precision="exact", normalize=True,
                                     check=True).cpu().numpy().reshape(Q, C)
    cpg = C // G
    for g in range(G):
        plan = mo.dense_to_csr_vectorized(shape, loc, wts, g)
        ref, _ = c_oracle.msda_c(np.ascontiguousarray(seen[:, g * cpg:(g + 1) * cpg]), tiles, 4, *plan)
        assert out[:, g * cpg:(g + 1) * cpg].tobytes() == ref.tobytes(), g


@pytest.mark.parametrize("cams,precision", [(2, "fast"), (6, "fast"), (6, "exact"), (6, "fast_h2")])
def test_dense_zero_weight_sum_raises(cuda_dev, cams, precision):
    """normalize=True with one (anchor, group) whose weights are all zero:
    every path (one camera group, split camera groups + normalising pass,
    exact) reports the zero sum; without normalisation the call succeeds and
    that group's channels are exactly zero."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(17)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=1, n_q=3, n_p=13, cams=cams, n_levels=4, groups=8,
                                                channels=256, size_lo=6, size_hi=20)
    wts[0, 1, ..., 5] = 0.0
    dt = torch.float16 if precision == "fast_h2" else torch.float32
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, dtype=dt)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    with pytest.raises(ValueError, match="sum to zero"):
        ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision=precision, normalize=True, check=True)
    out = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision=precision, normalize=False,
                                     check=True).cpu().numpy()
    assert not out[0, 1, 5 * 32:6 * 32].any()
    assert np.isfinite(out).all()


@pytest.mark.parametrize("cams,levels,dt", [
    (6, [(64, 176), (32, 88), (16, 44), (8, 22)], "float32"),      # cfg1 (f32 staged coarse levels)
    (16, [(270, 480), (135, 240), (68, 120), (34, 60)], "float32"),  # cfg2 shape: 4 camera groups, maps >> L2
    (32, [(64, 176), (32, 88), (16, 44), (8, 22)], "bfloat16"),    # cfg4 MSDA part (staged coarse levels)
    (64, [(64, 176), (32, 88), (16, 44), (8, 22)], "float16")])    # cfg3 per layer (staged coarse levels)
@pytest.mark.parametrize("normalize", [True, False])
def test_dense_full_size_vs_c_oracle(c_oracle, cuda_dev, cams, levels, dt, normalize):
    """BASELINE shapes at full size (900 anchors, 13 points, C = 256, G = 8),
    normalised, each path against the per-group C oracle (SURVEY §8(c):
    msda_reference on each group's channel slice) on the features the GPU
    reads: EXACT bit for bit; FAST (f32 products, any order: the camera
    groups' and levels' partial sums are red.add-ed) 1e-4 of max|ref|;
    FAST_H2 (half2 products and partials, f16) the north_star's 1e-2."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(97 + cams)
    C, G, Q, P = 256, 8, 900, 13
    dtype = getattr(torch, dt)
    n_rows = cams * sum(h * w for h, w in levels)
    table = (torch.rand((1, n_rows, C), generator=torch.Generator().manual_seed(cams)) * 2 - 1).to(cuda_dev, dtype)
    shape = np.array([levels] * cams, dtype=np.int32)
    start = np.cumsum([0] + [h * w for _ in range(cams) for h, w in levels])[:-1].reshape(cams, 4)
    feats = ops.DeviceFeatures(table, torch.from_numpy(shape), torch.from_numpy(start.astype(np.int64)))
    loc_np = rng.uniform(-0.02, 1.02, (1, Q, P, cams, 2)).astype(np.float32)
    logits = torch.from_numpy(rng.standard_normal((1, Q, P * cams * 4, G)).astype(np.float32)).to(cuda_dev)
    wts = torch.softmax(logits, dim=2).reshape(1, Q, P, cams, 4, G).contiguous()
    loc = torch.from_numpy(loc_np).to(cuda_dev)
    seen = feats.table[0].float().cpu().numpy()
    tiles = [(int(start[c, m]), h, w) for c in range(cams) for m, (h, w) in enumerate(levels)]
    ref = c_oracle.msda_dense_groups_c(seen, tiles, shape, loc_np, wts.cpu().numpy(), 4, normalize=normalize)
    del seen
    scale = float(np.abs(ref).max())
    exact = ops.deformable_aggregation(feats, None, None, loc, wts, precision="exact", normalize=normalize,
                                       check=True)
    assert exact.cpu().numpy().tobytes() == ref.tobytes()
    fast = ops.deformable_aggregation(feats, None, None, loc, wts, precision="fast", normalize=normalize,
                                      check=True)
    assert float(np.abs(fast.cpu().numpy() - ref).max()) <= 1e-4 * scale
    if dt == "float16":
        h2 = ops.deformable_aggregation(feats, None, None, loc, wts, precision="fast_h2", normalize=normalize,
                                        check=True)
        assert float(np.abs(h2.cpu().numpy() - ref).max()) <= 1e-2 * max(1.0, scale)


@pytest.mark.parametrize("dt,precision,normalize", [("float32", "exact", True), ("float16", "exact", False),
                                                    ("float32", "fast", True), ("float16", "fast_h2", False),
                                                    ("bfloat16", "fast", True), ("bfloat16", "exact", False)])
def test_dense_run_to_run(cuda_dev, dt, precision, normalize):
    """Determinism contract: EXACT is run-to-run
    bit-identical (one sequential chain per (query, channel)); FAST / FAST_H2
    add camera-group and level partials with red.add in whatever order the
    CTAs finish, so two calls agree to the FAST tolerance, not to the bit."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(41)
    cams, levels, C, G, Q, P = 12, [(64, 176), (32, 88), (16, 44), (8, 22)], 256, 8, 300, 13
    n_rows = cams * sum(h * w for h, w in levels)
    table = (torch.rand((1, n_rows, C), generator=torch.Generator().manual_seed(5)) * 2 - 1).to(cuda_dev,
                                                                                                getattr(torch, dt))
    shape = np.array([levels] * cams, dtype=np.int32)
    start = np.cumsum([0] + [h * w for _ in range(cams) for h, w in levels])[:-1].reshape(cams, 4)
    feats = ops.DeviceFeatures(table, torch.from_numpy(shape), torch.from_numpy(start.astype(np.int64)))
    loc = torch.from_numpy(rng.uniform(0, 1, (1, Q, P, cams, 2)).astype(np.float32)).to(cuda_dev)
    wts = torch.from_numpy(rng.uniform(0.01, 1, (1, Q, P, cams, 4, G)).astype(np.float32)).to(cuda_dev)
    outs = [ops.deformable_aggregation(feats, None, None, loc, wts, precision=precision, normalize=normalize,
                                       check=True).cpu().numpy() for _ in range(3)]
    if precision == "exact":
        assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()
    else:
        tol = (1e-2 if precision == "fast_h2" else 1e-5) * float(np.abs(outs[0]).max())
        assert float(np.abs(outs[0] - outs[1]).max()) <= tol and float(np.abs(outs[0] - outs[2]).max()) <= tol


@pytest.mark.parametrize("dt", ["float16", "bfloat16"])
def test_dense_batched_scenes_vs_c_oracle(c_oracle, cuda_dev, dt):
    """Four scenes of 32 cameras in one call (the cfg5 stream-sharded shape on
    a smaller batch): 3,600 anchors, so the fine-level gather keeps its long
    104-sample chains and the staged kernel's anchor chunks span whole
    scenes — FAST and (f16) FAST_H2 against the C oracle per scene."""
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(404)
    bs, cams, C, G, Q, P = 4, 32, 256, 8, 900, 13
    levels = [(64, 176), (32, 88), (16, 44), (8, 22)]
    dtype = getattr(torch, dt)
    n_rows = cams * sum(h * w for h, w in levels)
    table = (torch.rand((bs, n_rows, C), generator=torch.Generator().manual_seed(5)) * 2 - 1).to(cuda_dev, dtype)
    shape = np.array([levels] * cams, dtype=np.int32)
    start = np.cumsum([0] + [h * w for _ in range(cams) for h, w in levels])[:-1].reshape(cams, 4)
    feats = ops.DeviceFeatures(table, torch.from_numpy(shape), torch.from_numpy(start.astype(np.int64)))
    loc_np = rng.uniform(0.0, 1.0, (bs, Q, P, cams, 2)).astype(np.float32)
    logits = torch.from_numpy(rng.standard_normal((bs, Q, P * cams * 4, G)).astype(np.float32)).to(cuda_dev)
    wts = torch.softmax(logits, dim=2).reshape(bs, Q, P, cams, 4, G).contiguous()
    w_np = wts.cpu().numpy()
    loc = torch.from_numpy(loc_np).to(cuda_dev)
    tiles = [(int(start[c, m]), h, w) for c in range(cams) for m, (h, w) in enumerate(levels)]
    precs = ["fast", "fast_h2"] if dt == "float16" else ["fast"]
    got = {p: ops.deformable_aggregation(feats, None, None, loc, wts, precision=p, check=True).cpu().numpy()
           for p in precs}
    for b in range(bs):
        seen = feats.table[b].float().cpu().numpy()
        ref = c_oracle.msda_dense_groups_c(seen, tiles, shape, loc_np[b:b + 1], w_np[b:b + 1], 4)[0]
        scale = float(np.abs(ref).max())
        assert float(np.abs(got["fast"][b] - ref).max()) <= 1e-4 * scale, b
        if "fast_h2" in got:
            assert float(np.abs(got["fast_h2"][b] - ref).max()) <= 1e-2 * max(1.0, scale), b
