"""GPU parity of the two SURVEY §8(f) components either side of the MSDA
path: feature painting (simulator.py:249-289) and the tracker's association
cost (tracker.py:105-142).  Oracles: the reference's own outputs
(tests/golden/paint.npz, assoc.npz) and oracle/scene_oracle.py (pinned to
them in test_oracle_golden.py).  Bar: bit-identical bytes (f64 cost
matrices; f32 painted tables given the reference's numpy background)."""

import numpy as np
import pytest

from test_oracle_golden import paint_scene_inputs

pytestmark = pytest.mark.gpu


def _scene(g, k, cuda_dev):
    from paper_2601_10819_b200 import ops

    seed, frame, C, sigs, strides, bgs = paint_scene_inputs(g, k)
    cams = ops.Cameras(g[f"K{k}"], g[f"R{k}"], g[f"t{k}"], device=cuda_dev)
    n_obj = len(g[f"ids{k}"])
    sig = np.array(sigs[:n_obj]) if n_obj else None
    background = np.concatenate([b.reshape(-1, C) for b in bgs])
    return cams, seed, frame, C, sig, n_obj, strides, background


def test_paint_matches_reference(golden, cuda_dev):
    import torch

    from paper_2601_10819_b200 import ops

    g = golden("paint")
    k = 0
    while f"seed{k}" in g:
        cams, seed, frame, C, sig, n_obj, strides, bg = _scene(g, k, cuda_dev)
        for dt in (torch.float32, torch.float16, torch.bfloat16):
            feats = ops.paint(cams, g[f"wh{k}"], strides, C, g[f"ent{k}"], n_obj, sig, background=bg, dtype=dt)
            got = feats.table[0].cpu()
            want = torch.from_numpy(g[f"table{k}"]).to(dt)  # the reference's f32 table, RNE to the storage dtype
            assert got.view(torch.uint8).numpy().tobytes() == want.view(torch.uint8).numpy().tobytes(), (k, dt)
        k += 1
    assert k == 3


def test_paint_feeds_msda(golden, cuda_dev):
    """The painted table is a DeviceFeatures the MSDA path consumes directly."""
    import torch

    from oracle import msda_oracle as mo
    from paper_2601_10819_b200 import ops

    g = golden("paint")
    cams, seed, frame, C, sig, n_obj, strides, bg = _scene(g, 1, cuda_dev)
    feats = ops.paint(cams, g["wh1"], strides, C, g["ent1"], n_obj, sig, background=bg)
    shape = feats.spatial_shape.cpu().numpy()
    n_cams, n_levels = shape.shape[:2]
    rng = np.random.default_rng(5)
    loc = rng.uniform(0, 1, (1, 20, 13, n_cams, 2)).astype(np.float32)
    w = rng.uniform(0.01, 1, (1, 20, 13, n_cams, n_levels, 2)).astype(np.float32)
    out = ops.deformable_aggregation(feats, None, None, torch.from_numpy(loc).to(cuda_dev),
                                     torch.from_numpy(w).to(cuda_dev), precision="exact", check=True)
    starts = feats.scale_start_index.cpu().numpy().reshape(-1)
    tiles = [(int(starts[i]), int(shape.reshape(-1, 2)[i, 0]), int(shape.reshape(-1, 2)[i, 1]))
             for i in range(n_cams * n_levels)]
    ref = mo.msda_dense_groups(g["table1"], tiles, shape, loc, w, n_levels)
    assert out.cpu().numpy().tobytes() == ref.tobytes()


def test_paint_device_background(golden, cuda_dev):
    """Without a host background the device draws N(0, sigma) (Philox):
    deterministic per (seed, frame), the right law, and the same painting."""
    from paper_2601_10819_b200 import ops

    g = golden("paint")
    cams, seed, frame, C, sig, n_obj, strides, bg = _scene(g, 1, cuda_dev)
    sigma = 0.05
    a = ops.paint(cams, g["wh1"], strides, C, g["ent1"], n_obj, sig, sigma=sigma, seed=seed, frame=frame)
    b = ops.paint(cams, g["wh1"], strides, C, g["ent1"], n_obj, sig, sigma=sigma, seed=seed, frame=frame)
    c = ops.paint(cams, g["wh1"], strides, C, g["ent1"], n_obj, sig, sigma=sigma, seed=seed, frame=frame + 1)
    ta, tb, tc = (x.table[0].cpu().numpy().astype(np.float64) for x in (a, b, c))
    assert ta.tobytes() == tb.tobytes() and ta.tobytes() != tc.tobytes()
    # which rows carry a signature: from the reference table vs its own background
    ref = g["table1"].astype(np.float64)
    winner = np.full(ref.shape[0], -1)
    for i in range(n_obj):
        hit = np.all(np.abs(ref - bg - sig[i]) < 1e-6, axis=1)
        winner[hit] = i
    noise = ta.copy()
    noise[winner >= 0] -= sig[winner[winner >= 0]]
    assert abs(noise.mean()) < 3 * sigma / np.sqrt(noise.size)
    assert abs(noise.std() / sigma - 1) < 0.02
    assert (winner >= 0).sum() > 100


def test_assoc_cost_matches_reference(golden, cuda_dev):
    from oracle import scene_oracle as so
    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.tracker import TrackerParams, associate

    g = golden("assoc")
    k = 0
    while f"qc{k}" in g:
        gate, ae, ag = (float(x) for x in g[f"par{k}"])
        cost, solver, adm = ops.association_cost(g[f"qc{k}"], g[f"dc{k}"], g[f"qe{k}"], g[f"de{k}"], gate, ae, ag,
                                                 device=cuda_dev)
        assert solver.cpu().numpy().tobytes() == g[f"solver{k}"].tobytes(), k
        c_ref, _, a_ref = so.association_cost(g[f"qc{k}"], g[f"dc{k}"], g[f"qe{k}"], g[f"de{k}"], gate, ae, ag)
        assert cost.cpu().numpy().tobytes() == c_ref.tobytes()
        assert np.array_equal(adm.cpu().numpy(), a_ref)
        # the whole association step (Hungarian on the host) against the reference's Assignment
        perm = np.random.default_rng(k).permutation(len(g[f"qids{k}"]))  # input order must not matter
        asg = associate(g[f"qids{k}"][perm], g[f"qc{k}"][perm], g[f"qe{k}"][perm], g[f"dc{k}"], g[f"de{k}"],
                        TrackerParams(gate, ae, ag), device=cuda_dev)
        assert np.array_equal(np.array(asg.matches, dtype=np.int64).reshape(-1, 2), g[f"matches{k}"])
        assert asg.total_cost == float(g[f"total{k}"])
        k += 1
    assert k == 4


@pytest.mark.parametrize("n_q,n_d,dim", [(300, 200, 128), (37, 45, 300), (5, 3, 7), (64, 64, 1024)])
def test_assoc_cost_large_and_odd_dims(cuda_dev, n_q, n_d, dim):
    """Tile edges, D < 8 (sequential sum), D > 128 (numpy's halving) against
    numpy's own np.linalg.norm — the reference's arithmetic."""
    from paper_2601_10819_b200 import ops

    rng = np.random.default_rng(n_q + dim)
    qc, dc = rng.uniform(-5, 5, (n_q, 3)), rng.uniform(-5, 5, (n_d, 3))
    qe, de = rng.standard_normal((n_q, dim)), rng.standard_normal((n_d, dim))
    cost, solver, adm = ops.association_cost(qc, dc, qe, de, 3.0, 0.5, 2.0, device=cuda_dev)
    geo = np.linalg.norm(qc[:, None, :] - dc[None, :, :], axis=2)
    emb = np.linalg.norm(qe[:, None, :] - de[None, :, :], axis=2)
    ref = 0.5 * emb + 2.0 * geo / 3.0
    assert cost.cpu().numpy().tobytes() == ref.tobytes()
    assert np.array_equal(adm.cpu().numpy(), geo <= 3.0)
    assert solver.cpu().numpy().tobytes() == np.where(geo <= 3.0, ref, 1e9).tobytes()
