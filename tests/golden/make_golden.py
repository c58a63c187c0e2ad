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
    out = {}
    for k, (cams, objs, vis, behind) in enumerate(scenes):
        out[f"K{k}"] = np.array([[c.focal_x, c.focal_y, c.principal_x, c.principal_y] for c in cams])
        out[f"R{k}"] = np.array([c.rotation for c in cams])
        out[f"t{k}"] = np.array([c.translation for c in cams])
        out[f"obj{k}"] = np.array(objs)
        out[f"vis{k}"] = vis
        out[f"behind{k}"] = behind
    return out


def main():
    jobs = [("visibility", visibility_case), ("fpyr", fpyr_case), ("crit1", crit1), ("features", features_cases), ("bench", bench_cases), ("dense", dense_cases),
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
