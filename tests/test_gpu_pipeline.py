"""End to end on the GPU: the components either side of the MSDA path
composed the way the reference's tracker loop uses them:

    paint_pyramids (simulator.py:249-315)     -> channel-last table (device)
    visible_fraction (visibility.py:46-115)   -> v_i per (camera, object)
    extract_view + fuse_or_memory (oae.py)    -> one embedding per object
    associate (tracker.py:105-142)            -> track <-> detection matches

Two frames of one scene are painted (background drawn with the reference's
numpy generator, so the tables are bit-identical to the reference's); the
frame-0 embeddings become track memories, the frame-1 embeddings detection
embeddings.  Every stage is checked against the CPU oracle fed the same
inputs, and the association must recover the identities."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ring(n, radius=9.0, height=3.5, focal=260.0, size=(704, 256)):
    Ks, Rs, ts = [], [], []
    for i in range(n):
        ang = 2 * math.pi * i / n + 0.3
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


def test_paint_visibility_oae_associate(cuda_dev):
    import torch

    from oracle import msda_oracle as mo
    from oracle import scene_oracle as so
    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.tracker import TrackerParams, associate

    seed, C, cams = 23, 128, 4
    strides = [8.0, 16.0, 32.0]
    K, R, T = _ring(cams)
    wh = [[704, 256]] * cams
    camd = ops.Cameras(K, R, T, device=cuda_dev)
    ids = [4, 9, 15]
    objs0 = np.array([[-1.5, 0.5, 0.9, 0.7, 0.7, 1.8, 0.2], [1.2, -1.0, 0.9, 0.8, 0.6, 1.7, -0.5],
                      [0.3, 2.0, 0.9, 0.6, 0.9, 1.9, 1.1]])
    occ = np.array([[0.0, -4.0, 1.2, 0.3, 2.5, 2.4, 0.0]])
    sig = np.array([so.identity_signature(seed, i, C) for i in ids])
    scene_frames = []
    for frame, shift in ((0, 0.0), (1, 0.15)):
        objs = objs0.copy()
        objs[:, 0] += shift  # the objects walk a little between frames
        ents = np.concatenate([objs, occ])
        scene = ops.PaintScene(camd, wh, strides, C, ents, len(ids), sig)
        shape = scene.shape_host.numpy()
        bgs, tiles, r = [], [], 0
        for c in range(cams):
            for m in range(len(strides)):
                h, w = shape[c, m]
                bgs.append(so.paint_background(seed, frame, c, m, 0.05, (h, w, C)))
                tiles.append((r, int(h), int(w)))
                r += int(h * w)
        feats = scene.run(background=np.concatenate([b.reshape(-1, C) for b in bgs]))
        # stage 1: painting, bit-identical to the oracle's restatement of the reference
        ref_tab = np.concatenate([so.paint_grid(K[c], R[c], T[c], wh[c], strides[m], ents, list(sig) + [None],
                                                bgs[c * len(strides) + m]).reshape(-1, C)
                                  for c in range(cams) for m in range(len(strides))])
        table = feats.table[0].cpu().numpy()
        assert table.tobytes() == ref_tab.tobytes()
        # stage 2: visibility of every object in every camera (occluders block)
        vis, behind = ops.visibility(camd, wh, ents, grid=64)
        vis = vis.cpu().numpy()[:, :len(ids)].T.copy()  # [objects, cams]
        assert not behind.cpu().numpy().any() and vis.max() > 0.5
        # stage 3: occlusion-aware pooling at the objects' boxes
        anchors = np.zeros((len(ids), 10), dtype=np.float32)
        anchors[:, :7] = objs
        offsets = np.random.default_rng(3).uniform(-1, 1, (6, 3)).astype(np.float32)
        desc = np.random.default_rng(4).standard_normal((len(ids), C)).astype(np.float32)
        mem = np.random.default_rng(5).standard_normal((len(ids), C)).astype(np.float32)
        mem /= np.linalg.norm(mem, axis=1, keepdims=True)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda_dev)  # noqa: E731
        emb, occl = ops.oae_pool(feats, t(anchors), offsets, camd, strides, t(desc), t(vis.astype(np.float32)),
                                 t(mem))
        emb = emb.cpu().numpy()
        for q in range(len(ids)):
            kps = mo.keypoints(anchors[q].astype(np.float64), offsets.astype(np.float64))
            views = [mo.extract_view(table, tiles, len(strides), c, strides, K[c], R[c], T[c], kps,
                                     desc[q].astype(np.float64)) for c in range(cams)]
            ref, ref_occ = mo.fuse(views, vis[q].astype(np.float32), mem[q])
            assert bool(occl[q]) == ref_occ
            assert np.abs(emb[q] - ref).max() <= 1e-4
        scene_frames.append((objs, emb.astype(np.float64)))
    # stage 4: tracks (frame 0) vs detections (frame 1)
    (c0, e0), (c1, e1) = scene_frames
    e0 /= np.linalg.norm(e0, axis=1, keepdims=True)
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    det_order = [2, 0, 1]  # detections arrive in another order
    params = TrackerParams(gate_radius=1.0, alpha_emb=1.0, alpha_geo=1.0)
    asg = associate(ids, c0[:, :3], e0, c1[det_order, :3], e1[det_order], params, device=cuda_dev)
    assert sorted(asg.matches) == sorted((ids[d], k) for k, d in enumerate(det_order))
    cost, _, _ = so.association_cost(c0[:, :3], c1[det_order, :3], e0, e1[det_order], 1.0, 1.0, 1.0)
    assert asg.total_cost == sum(float(cost[ids.index(tid), d]) for tid, d in asg.matches)
