"""Generate the golden fixtures by running the REAL reference (mvtrack3d).

Run in the dev container (the reference is not available on the GPU box):

    python tests/golden/make_golden.py

It imports ``mvtrack3d`` from ``$MVTRACK3D_REF`` or ``/root/reference/pkg/src``
and writes ``tests/golden/*.npz``.  The tests regenerate the same inputs from
the same seeds (tests/helpers.py) and compare against these outputs, so the
fixtures hold outputs plus an input digest, not the inputs themselves.
"""

from __future__ import annotations

import math
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, os.environ.get("MVTRACK3D_REF", "/root/reference/pkg/src"))

from mvtrack3d import features as F  # noqa: E402
from mvtrack3d import geometry as G  # noqa: E402
from mvtrack3d import oae as O  # noqa: E402
from mvtrack3d.bench import BenchWorkload, generate_workload  # noqa: E402

import helpers  # noqa: E402


def ref_pyramids(grids, n_cams, n_levels):
    pyrs = []
    for cam in range(n_cams):
        lv = [F.FeatureGrid(stride=4.0 * 2 ** m, values=grids[(cam, m)]) for m in range(n_levels)]
        pyrs.append(F.FeaturePyramid(cam, lv))
    return pyrs


def crit1(n=10_000):
    """Criterion-1 workloads (seed 2024): reference FULL and PACKED_HALF outputs."""
    rng = np.random.default_rng(2024)
    full, half, lens, digests = [], [], [], []
    for i in range(n):
        grids, n_cams, n_levels, per_query = helpers.tiny_workload(rng)
        pyrs = ref_pyramids(grids, n_cams, n_levels)
        plan = F.SamplePlan(per_query)
        ref, _ = F.msda_reference(pyrs, plan)
        hf, _ = F.msda_optimized(pyrs, plan, precision=F.PrecisionMode.PACKED_HALF, workers=(1, 2, 4)[i % 3])
        full.append(ref.reshape(-1))
        half.append(hf.reshape(-1))
        lens.append(ref.size)
        digests.append(helpers.per_query_hash(per_query))
    import hashlib

    return dict(full=np.concatenate(full), half=np.concatenate(half), lens=np.array(lens, dtype=np.int64),
                input_digest=np.array(hashlib.sha256("".join(digests).encode()).hexdigest()))


def features_cases():
    """test_features.py-style random cases (seeds 7, 9, 10, 13 shapes)."""
    out = {}
    rng = np.random.default_rng(7)
    fulls, halves, lens = [], [], []
    for i in range(60):
        n_cams, n_levels = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        channels = int(rng.choice([2, 4, 8, 16]))
        grids, _ = helpers.make_pyramids(rng, n_cams=n_cams, n_levels=n_levels, channels=channels)
        per_query = helpers.make_plan(rng, grids, n_queries=int(rng.integers(1, 9)))
        if i % 7 == 3:
            per_query.insert(1, [])  # an empty query in the middle
        pyrs = ref_pyramids(grids, n_cams, n_levels)
        plan = F.SamplePlan(per_query)
        ref, emp = F.msda_reference(pyrs, plan)
        hf, _ = F.msda_optimized(pyrs, plan, precision=F.PrecisionMode.PACKED_HALF)
        un, _ = F.msda_reference(pyrs, plan, normalize=False)
        fulls.append(np.concatenate([ref.reshape(-1), un.reshape(-1)]))
        halves.append(hf.reshape(-1))
        lens.append(ref.size)
    out["full"] = np.concatenate(fulls)
    out["half"] = np.concatenate(halves)
    out["lens"] = np.array(lens, dtype=np.int64)
    return out


def bench_cases():
    """Reference bench workloads: checksums (+ outputs for the small ones)."""
    out = {}
    small = BenchWorkload(cameras=2, levels=2, channels=8, queries=16, points_per_query=4, level0_size=(8, 8))
    med = BenchWorkload(cameras=3, levels=4, channels=32, queries=40, points_per_query=13, level0_size=(32, 88))
    for name, wl in (("small", small), ("medium", med)):
        pyrs, plan, ck = generate_workload(wl)
        ref, _ = F.msda_reference(pyrs, plan)
        hf, _ = F.msda_optimized(pyrs, plan, precision=F.PrecisionMode.PACKED_HALF)
        out[f"{name}_checksum"] = np.array(ck)
        out[f"{name}_full"] = ref
        out[f"{name}_half"] = hf
    for name, wl in (("default", BenchWorkload()),
                     ("cfg1", BenchWorkload(cameras=6, level0_size=(64, 176))),
                     ("cfg2", BenchWorkload(cameras=16, level0_size=(270, 480)))):
        t0 = time.time()
        _, _, ck = generate_workload(wl)
        out[f"{name}_checksum"] = np.array(ck)
        print(f"  {name} checksum in {time.time() - t0:.1f}s")
    return out


def dense_cases():
    """Sparse4D dense layout with groups → per-group reference msda_reference."""
    rng = np.random.default_rng(31)
    outs = []
    for i in range(6):
        groups = (1, 2, 4)[i % 3]
        grids, shape, loc, wts = helpers.make_dense(rng, bs=1 + i % 2, n_q=4, n_p=3, cams=2, n_levels=2,
                                                    groups=groups, channels=8)
        bs, n_q, n_p, cams, _ = loc.shape
        n_levels = shape.shape[1]
        c_n = 8
        cg = c_n // groups
        res = np.zeros((bs * n_q, c_n), dtype=np.float32)
        for normalize in (False, True):
            for g in range(groups):
                per_query = []
                for b in range(bs):
                    for q in range(n_q):
                        s = []
                        for p in range(n_p):
                            for c in range(cams):
                                x, y = loc[b, q, p, c]
                                for m in range(n_levels):
                                    h, w = shape[c, m]
                                    uu = np.float32(np.float32(x * np.float32(w)) - np.float32(0.5))
                                    vv = np.float32(np.float32(y * np.float32(h)) - np.float32(0.5))
                                    s.append((c, m, float(uu), float(vv), float(wts[b, q, p, c, m, g])))
                        per_query.append(s)
                sub = {k: np.ascontiguousarray(v[:, :, g * cg:(g + 1) * cg]) for k, v in grids.items()}
                pyrs = ref_pyramids(sub, cams, n_levels)
                r, _ = F.msda_reference(pyrs, F.SamplePlan(per_query), normalize=normalize)
                res[:, g * cg:(g + 1) * cg] = r
            outs.append(res.copy().reshape(-1))
    return {"out": np.concatenate(outs)}


def ring_cameras(n, radius=12.0, height=4.0, focal=300.0, size=(704, 256)):
    cams = []
    for i in range(n):
        ang = 2 * math.pi * i / n
        pos = (radius * math.cos(ang), radius * math.sin(ang), height)
        cams.append(G.camera_looking_at(pos, (0.0, 0.0, 0.9), focal, (size[0] / 2, size[1] / 2), size))
    return cams


def projection_cases():
    """generate_keypoints → motion_compensate → project_point goldens (f64)."""
    rng = np.random.default_rng(41)
    cams = ring_cameras(5)
    rows = []
    offsets = rng.uniform(-1, 1, size=(6, 3))
    anchors = []
    for _ in range(12):
        a = [rng.uniform(-4, 4), rng.uniform(-4, 4), 0.9, 0.6, 0.6, 1.8, rng.uniform(-math.pi, math.pi),
             rng.uniform(-1, 1), rng.uniform(-1, 1), 0.0]
        anchors.append(a)
        st = G.ObjectState3D(*a)
        kp = G.motion_compensate(G.generate_keypoints(st, offsets), st.velocity, 0.5)
        for ci, cam in enumerate(cams):
            for p, pt in enumerate(kp.points):
                try:
                    u, v, d = G.project_point(cam, pt)
                    rows.append((ci, p, u, v, d))
                except Exception:
                    rows.append((ci, p, np.nan, np.nan, np.nan))
    camK = np.array([[c.focal_x, c.focal_y, c.principal_x, c.principal_y] for c in cams])
    camR = np.array([c.rotation for c in cams])
    camT = np.array([c.translation for c in cams])
    return {"anchors": np.array(anchors), "offsets": offsets, "K": camK, "R": camR, "t": camT,
            "proj": np.array(rows, dtype=np.float64)}


def oae_cases():
    """extract_view_feature + fuse_or_memory on a small ring scene."""
    rng = np.random.default_rng(43)
    n_cams, n_levels, channels = 4, 3, 16
    cams = ring_cameras(n_cams, size=(128, 64), focal=80.0)
    strides = [8.0, 16.0, 32.0]
    grids = {}
    for c in range(n_cams):
        for m, s in enumerate(strides):
            h, w = int(math.ceil(64 / s)), int(math.ceil(128 / s))
            grids[(c, m)] = rng.standard_normal((h, w, channels)).astype(np.float32)
    pyrs = [F.FeaturePyramid(c, [F.FeatureGrid(stride=s, values=grids[(c, m)]) for m, s in enumerate(strides)])
            for c in range(n_cams)]
    offsets = rng.uniform(-1, 1, size=(6, 3))
    anchors, desc, vis, mem, embs, occl, views = [], [], [], [], [], [], []
    for qi in range(10):
        a = [rng.uniform(-3, 3), rng.uniform(-3, 3), 0.9, 0.6, 0.6, 1.8, rng.uniform(-math.pi, math.pi), 0.0, 0.0, 0.0]
        st = G.ObjectState3D(*a)
        kp = G.generate_keypoints(st, offsets)
        d = rng.standard_normal(channels)
        memory = O.Embedding.normalize(rng.standard_normal(channels))
        v = rng.uniform(0.0, 1.0, size=n_cams)
        if qi == 3:
            v[:] = 1e-4  # all occluded → memory fallback
        query = O.Query(track_id=qi, anchor=st, memory=memory, descriptor=d)
        pv = [O.extract_view_feature(pyrs[c], cams[c], kp, query) for c in range(n_cams)]
        e = O.fuse_or_memory(pv, list(v), memory)
        anchors.append(a)
        desc.append(d)
        vis.append(v)
        mem.append(memory.values)
        embs.append(e.values)
        views.append(np.array([x[0] for x in pv]))
        occl.append(e is memory)
    return {"grids": np.concatenate([grids[(c, m)].reshape(-1) for c in range(n_cams) for m in range(n_levels)]),
            "shapes": np.array([grids[(c, m)].shape[:2] for c in range(n_cams) for m in range(n_levels)]),
            "strides": np.array(strides), "K": np.array([[c.focal_x, c.focal_y, c.principal_x, c.principal_y] for c in cams]),
            "R": np.array([c.rotation for c in cams]), "t": np.array([c.translation for c in cams]),
            "offsets": offsets, "anchors": np.array(anchors), "desc": np.array(desc), "vis": np.array(vis),
            "memory": np.array(mem), "emb": np.array(embs), "occluded": np.array(occl), "views": np.array(views)}


def fpyr_case():
    """A small FPYR container written by the reference writer."""
    import tempfile

    from mvtrack3d.simulator import write_pyramid_sequence

    rng = np.random.default_rng(47)
    frames = []
    for f in range(3):
        frame = {}
        for cam in (7, 2):  # unsorted ids: the container sorts them
            lv = [F.FeatureGrid(stride=8.0 * 2 ** m, values=rng.standard_normal((5 - m, 6 - m, 4)).astype(np.float32))
                  for m in range(2)]
            frame[cam] = F.FeaturePyramid(cam, lv)
        frames.append(frame)
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "pyr.bin"
        write_pyramid_sequence(path, frames)
        blob = np.frombuffer(path.read_bytes(), dtype=np.uint8)
    return {"blob": blob}


def visibility_case():
    """visible_fraction for every (camera, object) of random ring scenes."""
    from mvtrack3d.visibility import visible_fraction

    rng = np.random.default_rng(53)
    scenes = []
    for k in range(4):
        cams = ring_cameras(3 + k, size=(640, 480), focal=400.0)
        objs = []
        for _ in range(6 + 2 * k):
            objs.append([rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(0.5, 1.5), rng.uniform(0.4, 1.5),
                         rng.uniform(0.4, 2.0), rng.uniform(0.8, 2.0), rng.uniform(-math.pi, math.pi)])
        if k == 1:
            objs.append([12.0 * math.cos(0.0), 0.0, 4.2, 0.5, 0.5, 0.5, 0.0])  # at camera 0: partly/fully behind
        states = [G.ObjectState3D(*o) for o in objs]
        vis = np.zeros((len(cams), len(states)))
        behind = np.zeros((len(cams), len(states)), dtype=bool)
        for ci, cam in enumerate(cams):
            for oi, st in enumerate(states):
                sc = visible_fraction(cam, st, states, grid=64)
                vis[ci, oi] = sc.value
                behind[ci, oi] = sc.fully_behind
        scenes.append((cams, objs, vis, behind))
    # denser scenes (more, larger, overlapping boxes; other image sizes): many
    # sample points fall near rect edges, where the projection's last bit decides
    rng2 = np.random.default_rng(54)
    for k in range(12):
        size = [(640, 480), (704, 256), (1920, 1080)][k % 3]
        cams = ring_cameras(2 + k % 5, size=size, focal=float(rng2.uniform(250, 900)), radius=float(rng2.uniform(6, 14)))
        objs = []
        for _ in range(10 + 2 * k):
            objs.append([rng2.uniform(-4, 4), rng2.uniform(-4, 4), rng2.uniform(0.3, 1.5), rng2.uniform(0.3, 2.5),
                         rng2.uniform(0.3, 3.0), rng2.uniform(0.5, 2.5), rng2.uniform(-math.pi, math.pi)])
        states = [G.ObjectState3D(*o) for o in objs]
        vis = np.zeros((len(cams), len(states)))
        behind = np.zeros((len(cams), len(states)), dtype=bool)
        for ci, cam in enumerate(cams):
            for oi, st in enumerate(states):
                sc = visible_fraction(cam, st, states, grid=64)
                vis[ci, oi] = sc.value
                behind[ci, oi] = sc.fully_behind
        scenes.append((cams, objs, vis, behind))
    out = {}
    for k, (cams, objs, vis, behind) in enumerate(scenes):
        out[f"K{k}"] = np.array([[c.focal_x, c.focal_y, c.principal_x, c.principal_y] for c in cams])
        out[f"R{k}"] = np.array([c.rotation for c in cams])
        out[f"t{k}"] = np.array([c.translation for c in cams])
        out[f"obj{k}"] = np.array(objs)
        out[f"vis{k}"] = vis
        out[f"behind{k}"] = behind
        out[f"wh{k}"] = np.array([[c.width, c.height] for c in cams])
    return out


def paint_case():
    """paint_pyramids (simulator.py:249-315) on three scenes: several cameras,
    walkers, occluders, a nearer-object-wins overlap; frame 1 of each."""
    from mvtrack3d.simulator import FeatureParams, SceneConfig, SceneObject, paint_pyramids, simulate_truth

    out = {}
    specs = [
        # (seed, cameras [(pos, target, focal, (W, H))], walkers [(id, waypoints, dims)], occluders, C, strides)
        (3, [([0.0, -8.0, 3.0], [0.0, 0.0, 1.0], 200.0, (320, 240)), ([8.0, 0.0, 3.0], [0.0, 0.0, 1.0], 180.0, (300, 200))],
         [(0, [[0.0, -2.0, 0.0, 0.875], [4.0, 2.0, 0.0, 0.875]], (0.6, 0.6, 1.75)),
          (5, [[0.0, 0.0, 1.0, 0.9], [4.0, 1.0, -2.0, 0.9]], (0.8, 0.7, 1.8))],
         [[0.0, -4.0, 1.25, 0.3, 3.0, 2.5, 0.0]], 8, (8.0, 16.0)),
        (11, [([0.0, -9.0, 4.0], [0.0, 0.0, 1.0], 250.0, (352, 128)), ([-6.0, -6.0, 3.0], [0.0, 0.0, 0.9], 220.0, (352, 128)),
              ([6.0, 6.0, 3.5], [0.0, 0.0, 0.9], 240.0, (352, 128))],
         [(1, [[0.0, 0.0, -4.0, 1.0]], (1.0, 1.0, 1.8)), (2, [[0.0, 0.0, 0.0, 1.0]], (3.0, 3.0, 2.4)),
          (7, [[0.0, 2.0, 1.0, 0.9], [5.0, -1.0, 1.0, 0.9]], (0.5, 0.5, 1.7))],
         [[1.5, -3.0, 1.0, 0.4, 2.0, 2.0, 0.3], [-2.0, 1.0, 1.0, 1.0, 1.0, 2.0, 1.1]], 16, (4.0, 8.0, 16.0, 32.0)),
        (29, [([0.0, -5.0, 2.0], [0.0, 0.0, 1.0], 450.0, (640, 360))],
         [(3, [[0.0, -1.0, 0.0, 0.9]], (0.6, 0.6, 1.75)), (4, [[0.0, 1.0, 0.5, 0.9]], (0.7, 0.6, 1.8))],
         [], 4, (16.0, 32.0)),
    ]
    for k, (seed, cams, walkers, occ, C, strides) in enumerate(specs):
        cameras = {ci: G.camera_looking_at(pos, tgt, f, (wh[0] / 2.0, wh[1] / 2.0), wh)
                   for ci, (pos, tgt, f, wh) in enumerate(cams)}
        objs = [SceneObject(category="person", identity=i, dims=d, waypoints=np.array(wp)) for i, wp, d in walkers]
        cfg = SceneConfig(seed=seed, frame_rate=10.0, duration=0.1, cameras=cameras, objects=objs,
                          occluders=[G.ObjectState3D(*o) for o in occ],
                          features=FeatureParams(channels=C, strides=strides, background_sigma=0.01), visibility_grid=8)
        ft = simulate_truth(cfg)[1]
        pyr = paint_pyramids(cfg, ft)
        ents = [[t.state.x, t.state.y, t.state.z, t.state.w, t.state.l, t.state.h, t.state.yaw] for t in ft.objects]
        ents += [list(o) for o in occ]
        out[f"seed{k}"] = np.array([seed, ft.frame_index, C], dtype=np.int64)
        out[f"ids{k}"] = np.array([t.identity for t in ft.objects], dtype=np.int64)
        out[f"n_occ{k}"] = np.array(len(occ))
        out[f"ent{k}"] = np.array(ents, dtype=float)
        out[f"strides{k}"] = np.array(strides, dtype=float)
        c_ids = sorted(cameras)
        out[f"K{k}"] = np.array([[cameras[c].focal_x, cameras[c].focal_y, cameras[c].principal_x,
                                  cameras[c].principal_y] for c in c_ids])
        out[f"R{k}"] = np.array([cameras[c].rotation for c in c_ids])
        out[f"t{k}"] = np.array([cameras[c].translation for c in c_ids])
        out[f"wh{k}"] = np.array([[cameras[c].width, cameras[c].height] for c in c_ids], dtype=np.int32)
        out[f"table{k}"] = np.concatenate([g.values.reshape(-1, C) for c in c_ids for g in pyr[c].levels])
    return out


def assoc_case():
    """The association cost of tracker.associate (tracker.py:105-142): the
    solver_cost matrix handed to linear_sum_assignment is captured, plus the
    resulting Assignment."""
    from mvtrack3d import tracker as T
    from mvtrack3d.oae import Embedding, Query

    captured = []
    real = T.linear_sum_assignment

    def capture(m):
        captured.append(np.array(m, copy=True))
        return real(m)

    T.linear_sum_assignment = capture
    out = {}
    rng = np.random.default_rng(61)
    try:
        for k, (n_q, n_d, D, gate) in enumerate([(7, 9, 16, 2.0), (30, 25, 128, 1.5), (12, 12, 128, float("inf")),
                                                 (40, 33, 64, 3.0)]):
            def unit(n):
                v = rng.standard_normal((n, D))
                return v / np.linalg.norm(v, axis=1, keepdims=True)

            qe, de = unit(n_q), unit(n_d)
            qc = rng.uniform(-5, 5, (n_q, 3))
            dc = np.concatenate([qc[: n_d // 2] + rng.normal(0, 0.5, (n_d // 2, 3)),
                                 rng.uniform(-5, 5, (n_d - n_d // 2, 3))])
            ids = rng.permutation(1000)[:n_q]
            queries = [Query(track_id=int(ids[i]), anchor=G.ObjectState3D(*qc[i], 0.6, 0.6, 1.7, 0.0),
                             memory=Embedding(qe[i]), descriptor=np.zeros(D)) for i in range(n_q)]
            dets = [T.Detection(state=G.ObjectState3D(*dc[j], 0.6, 0.6, 1.7, 0.0), embedding=Embedding(de[j]),
                                confidence=1.0) for j in range(n_d)]
            params = T.TrackerParams(gate_radius=gate, alpha_emb=0.7 + 0.1 * k, alpha_geo=1.3 - 0.2 * k)
            asg = T.associate(T.QueryBank(queries=queries), dets, params)
            order = np.argsort(ids, kind="stable")  # the reference sorts queries by track id
            out[f"qc{k}"], out[f"dc{k}"] = qc[order], dc
            out[f"qe{k}"], out[f"de{k}"] = qe[order], de
            out[f"par{k}"] = np.array([gate, params.alpha_emb, params.alpha_geo])
            out[f"solver{k}"] = captured[-1]
            out[f"matches{k}"] = np.array(asg.matches, dtype=np.int64).reshape(-1, 2)
            out[f"total{k}"] = np.array(asg.total_cost)
            out[f"qids{k}"] = ids[order]
    finally:
        T.linear_sum_assignment = real
    return out


def bilinear_case():
    """The reference's own bilinear_sample (features.py:184-219) on random
    grids at random, integer, edge and out-of-grid cell coordinates
    (helpers.bilinear_inputs regenerates the inputs from the seed)."""
    grids, coords = helpers.bilinear_inputs(np.random.default_rng(71))
    out = {}
    for k, (grid, (us, vs)) in enumerate(zip(grids, coords)):
        pyr = F.FeaturePyramid(0, [F.FeatureGrid(stride=4.0, values=grid)])
        out[f"out{k}"] = np.stack([F.bilinear_sample(pyr, 0, float(u), float(v)) for u, v in zip(us, vs)])
    return out


def main():
    jobs = [("bilinear", bilinear_case), ("paint", paint_case), ("assoc", assoc_case), ("visibility", visibility_case), ("fpyr", fpyr_case), ("crit1", crit1), ("features", features_cases), ("bench", bench_cases), ("dense", dense_cases),
            ("projection", projection_cases), ("oae", oae_cases)]
    only = set(sys.argv[1:])
    for name, fn in jobs:
        if only and name not in only:
            continue
        t0 = time.time()
        data = fn()
        np.savez_compressed(HERE / f"{name}.npz", **data)
        print(f"{name}: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
