"""Edge shapes through every device entry point: empty inputs, single
camera / level / point, many groups, batch > 1, channel counts at the
kernel-selection boundaries.  Each result is checked against the oracle (or
for empty inputs, that nothing is written and nothing fails)."""

import numpy as np
import pytest

import helpers
from oracle import msda_oracle as mo

pytestmark = pytest.mark.gpu


def _feats(ops, torch, grids, shape, dev, dtype=None, batch=1):
    cams, n_levels = shape.shape[:2]
    table, tiles = mo.pack_grids(grids, cams, n_levels)
    start = np.array([t[0] for t in tiles], dtype=np.int64).reshape(cams, n_levels)
    tt = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(table, (batch,) + table.shape))).to(dev)
    if dtype is not None:
        tt = tt.to(dtype)
    return ops.DeviceFeatures(tt.contiguous(), torch.from_numpy(shape), torch.from_numpy(start)), table, tiles


@pytest.mark.parametrize("bs,q,p,cams,levels,groups,channels", [
    (1, 1, 1, 1, 1, 1, 2), (2, 3, 1, 1, 1, 2, 4), (1, 5, 2, 1, 3, 8, 256), (3, 2, 13, 2, 1, 32, 256),
    (1, 4, 3, 3, 2, 4, 128), (2, 2, 5, 2, 2, 16, 512)])
@pytest.mark.parametrize("precision", ["fast", "exact"])
def test_dense_edge_shapes(cuda_dev, bs, q, p, cams, levels, groups, channels, precision):
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(bs * 1000 + q * 100 + p * 10 + cams + groups)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=bs, n_q=q, n_p=p, cams=cams, n_levels=levels, groups=groups,
                                                channels=channels, size_lo=1, size_hi=7)
    feats, table, tiles = _feats(ops, torch, grids, shape, cuda_dev, batch=bs)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    for normalize in (False, True):
        out = ops.deformable_aggregation(feats, None, None, t(loc), t(wts), precision=precision, normalize=normalize,
                                         check=True).cpu().numpy()
        ref = mo.msda_dense_groups(table, tiles, shape, loc, wts, levels, normalize=normalize)
        if precision == "exact":
            assert out.tobytes() == ref.tobytes()
        else:
            assert np.abs(out - ref).max() <= 1e-4 * max(1e-12, np.abs(ref).max())


def test_empty_inputs_everywhere(cuda_dev):
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(5)
    grids, shape = helpers.make_pyramids(rng, n_cams=2, n_levels=2, channels=256)
    feats, table, tiles = _feats(ops, torch, {k: v for k, v in grids.items()}, np.array(
        [[[g.shape[0], g.shape[1]] for g in (grids[(c, 0)], grids[(c, 1)])] for c in range(2)], dtype=np.int32),
        cuda_dev)
    z = lambda *s, dt=torch.float32: torch.zeros(s, dtype=dt, device=cuda_dev)  # noqa: E731
    # CSR: zero queries, and queries without samples
    out, empty = ops.msda_csr(feats, torch.zeros(1, dtype=torch.int64, device=cuda_dev), z(0, dt=torch.int32),
                              z(0, dt=torch.int32), z(0), z(0), z(0))
    assert out.shape == (0, 256) and empty.numel() == 0
    for prec in ("exact", "fast"):
        out, empty = ops.msda_csr(feats, torch.zeros(4, dtype=torch.int64, device=cuda_dev), z(0, dt=torch.int32),
                                  z(0, dt=torch.int32), z(0), z(0), z(0), precision=prec)
        assert not out.cpu().numpy().any() and empty.cpu().numpy().all()
    # dense with zero anchors
    out = ops.deformable_aggregation(feats, None, None, z(1, 0, 3, 2, 2), z(1, 0, 3, 2, 2, 8), check=True)
    assert out.shape == (1, 0, 256)
    # association with an empty side
    cost, solver, adm = ops.association_cost(np.zeros((0, 3)), np.zeros((5, 3)), np.zeros((0, 16)),
                                             np.zeros((5, 16)), device=cuda_dev)
    assert cost.shape == (0, 5)
    # painting with no entities: background only
    K = np.array([[100.0, 100.0, 32.0, 16.0]])
    cams = ops.Cameras(K, np.eye(3).reshape(1, 9), np.zeros((1, 3)), device=cuda_dev)
    bg = rng.standard_normal((32 + 8, 4))  # 4 x 8 cells at stride 8, 2 x 4 at stride 16
    f = ops.paint(cams, [[64, 32]], [8.0, 16.0], 4, np.zeros((0, 7)), 0, None, background=bg)
    assert f.table[0].cpu().numpy().tobytes() == bg.astype(np.float32).tobytes()


def test_oae_and_projection_with_zero_queries(cuda_dev):
    import torch

    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(8)
    grids, _ = helpers.make_pyramids(rng, n_cams=1, n_levels=2, channels=8)
    shape = np.array([[[grids[(0, m)].shape[0], grids[(0, m)].shape[1]] for m in range(2)]], dtype=np.int32)
    feats, _, _ = _feats(ops, torch, grids, shape, cuda_dev)
    cams = ops.Cameras([[100.0, 100.0, 8.0, 8.0]], np.eye(3).reshape(1, 9), [[0.0, 0.0, 5.0]], device=cuda_dev)
    z = lambda *s: torch.zeros(s, device=cuda_dev)  # noqa: E731
    emb, occl = ops.oae_pool(feats, z(0, 10), np.zeros((0, 3), np.float32), cams, [4.0, 8.0], z(0, 8), z(0, 1),
                             z(0, 8))
    assert emb.shape == (0, 8) and occl.numel() == 0
    out = ops.msda_dense_project(feats, z(1, 0, 10), np.zeros((0, 3), np.float32), cams, [4.0, 8.0],
                                 z(1, 0, 7, 1, 2, 2), check=True)
    assert out.shape == (1, 0, 8)
