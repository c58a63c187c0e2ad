#!/usr/bin/env python
"""Per-path GPU timings for the non-headline BASELINE configs (dense Sparse4D
API, fused projection, OAE pooling).  bench.py holds the driver contract; this
tool prints one JSON line per config for DESIGN.md / profiles/.

Synthetic inputs per SURVEY §8(d): features U[-1, 1) channel-last,
sampling_location U[0, 1)^2 per (b, q, p, cam) shared across levels, weights
softmax over (P*cams*L) of N(0, 1) logits per (b, q, g), G = 8.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2601_10819_b200 import ops  # noqa: E402

from tools.sparse4d_cases import CFG1_LEVELS, CFG2_LEVELS, L2_BYTES as L2, make_dense_inputs  # noqa: E402
from tools.sparse4d_cases import make_feats as _make_feats, touched_bytes  # noqa: E402


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text())["hbm_gbs"] if p.exists() else 6650.0


def make_feats(cams, levels, C, dtype, dev, bs=1):
    return _make_feats(cams, levels, C, dtype, dev, bs=bs, seed=0)


def l2_ceiling():
    """Measured L2 -> SM random-row gather ceiling (tools/gather_ceiling.cu)."""
    p = ROOT / "profiles" / "r1" / "gather_ceiling.txt"
    best = None
    if p.exists():
        for line in p.read_text().splitlines():
            if line.startswith("pipe_") and "moved" in line:
                v = float(line.split("moved")[1].split("GB/s")[0])
                best = v if best is None else max(best, v)
    return best


def time_fn(fn, reps, flush):
    """Per-call CUDA-event times (ms), enqueued back to back without host
    synchronisation (as bench.py's sparse4d block): a host sync per call would
    add the host launch latency (~35 us per split dense call) to the device
    time.  ``flush`` rewrites a 2x-L2 buffer before every call (cold)."""
    scratch = torch.empty(2 * L2 // 4, device="cuda") if flush else None
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        if flush:
            scratch.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    return ts[len(ts) // 2], ts[0]


def dense_case(name, cams, levels, C, G, dtype, precision, reps, dev, Q=900, P=13, bs=1):
    feats = make_feats(cams, levels, C, dtype, dev, bs)
    loc, w = make_dense_inputs(bs, Q, P, cams, len(levels), G, dev)
    out = torch.empty((bs, Q, C), device=dev)
    esize = torch.finfo(dtype).bits // 8
    table_bytes = feats.table.numel() * esize
    fn = lambda: ops.deformable_aggregation(feats, None, None, loc, w, precision=precision, out=out)  # noqa: E731
    med, best = time_fn(fn, reps, flush=table_bytes < 2 * L2)
    tb, moved = touched_bytes(feats, loc, esize)
    alg = tb + loc.numel() * 4 + w.numel() * 4 + out.numel() * 4
    gbs = alg / (med / 1e3) / 1e9
    l2_gbs = moved / (med / 1e3) / 1e9
    ceil = l2_ceiling()
    cams_total = bs * cams
    return {"config": name, "path": "deformable_aggregation", "precision": precision, "dtype": str(dtype),
            "cams": cams, "groups": G, "latency_us": med * 1e3, "best_us": best * 1e3,
            "algorithmic_bytes": alg, "touched_feature_bytes": tb, "achieved_gbs": gbs, "frac": gbs / peak(),
            "camera_frames_per_s": cams_total / (med / 1e3),
            "streams_at_30fps_6layers": int(cams_total / (30 * 6 * med / 1e3)),
            "l2": "flushed" if table_bytes < 2 * L2 else "table > L2",
            "l2_gather": {"bytes": moved, "achieved_gbs": l2_gbs, "ceiling_gbs": ceil,
                          "frac": (l2_gbs / ceil) if ceil else None}}


def ring(cams, radius=12.0, height=4.0, focal=300.0, size=(704, 256)):
    import numpy as np

    Ks, Rs, ts = [], [], []
    for i in range(cams):
        ang = 2 * math.pi * i / cams
        pos = np.array([radius * math.cos(ang), radius * math.sin(ang), height])
        z = np.array([0.0, 0.0, 0.9]) - pos
        z /= np.linalg.norm(z)
        x = np.cross(z, [0.0, 0.0, 1.0])
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R = np.vstack([x, y, z])
        Ks.append([focal, focal, size[0] / 2, size[1] / 2])
        Rs.append(R)
        ts.append(-R @ pos)
    return np.array(Ks), np.array(Rs), np.array(ts)


def anchors_for(Q, dev, seed=2):
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = torch.zeros((Q, 10))
    a[:, 0:2] = torch.rand((Q, 2), generator=g) * 8 - 4
    a[:, 2] = 0.9
    a[:, 3:6] = torch.tensor([0.6, 0.6, 1.8])
    a[:, 6] = torch.rand(Q, generator=g) * 2 * math.pi - math.pi
    return a.to(dev)


def project_case(reps, dev, cams=6, C=256, G=8, Q=900):
    feats = make_feats(cams, CFG1_LEVELS, C, torch.float32, dev)
    K, R, T = ring(cams)
    camd = ops.Cameras(K, R, T, device=dev)
    anchors = anchors_for(Q, dev).unsqueeze(0)
    offs = (torch.rand((6, 3), generator=torch.Generator().manual_seed(3)) * 2 - 1).to(dev)
    strides = torch.tensor([4.0, 8.0, 16.0, 32.0], device=dev)  # resident: no per-call host copies
    _, w = make_dense_inputs(1, Q, 13, cams, 4, G, dev)
    out = torch.empty((1, Q, C), device=dev)
    fn = lambda: ops.msda_dense_project(feats, anchors, offs, camd, strides, w, dt=0.1, out=out)  # noqa: E731
    med, best = time_fn(fn, reps, flush=True)
    return {"config": "cfg1-project", "path": "msda_dense_project (fused keypoints + projection)",
            "precision": "fast", "dtype": "float32", "cams": cams, "latency_us": med * 1e3, "best_us": best * 1e3,
            "camera_frames_per_s": cams / (med / 1e3)}


def oae_case(reps, dev, cams=32, C=256, Q=900):
    feats = make_feats(cams, CFG1_LEVELS, C, torch.bfloat16, dev)
    K, R, T = ring(cams)
    camd = ops.Cameras(K, R, T, device=dev)
    anchors = anchors_for(Q, dev)
    offs = (torch.rand((6, 3), generator=torch.Generator().manual_seed(3)) * 2 - 1).to(dev)
    strides = torch.tensor([4.0, 8.0, 16.0, 32.0], device=dev)  # resident: no per-call host copies
    g = torch.Generator(device=dev).manual_seed(4)
    desc = torch.randn((Q, C), generator=g, device=dev)
    vis = torch.rand((Q, cams), generator=g, device=dev)
    mem = torch.nn.functional.normalize(torch.randn((Q, C), generator=g, device=dev), dim=1)
    fn = lambda: ops.oae_pool(feats, anchors, offs, camd, strides, desc, vis, mem, check=False)  # noqa: E731
    med, best = time_fn(fn, reps, flush=False)
    return {"config": "cfg4-oae", "path": "oae_pool (keypoint sampling + softmax + visibility fusion)",
            "dtype": "bfloat16", "cams": cams, "latency_us": med * 1e3, "best_us": best * 1e3,
            "queries_per_s": Q / (med / 1e3)}


def frame_case(reps, dev, cams=64, C=256, G=8, Q=900, P=13, layers=6, precision="fast_h2"):
    """The paper headline (BASELINE configs[2]): one frame of 64 fp16 camera
    streams through 6 decoder layers of MSDA — 6 deformable_aggregation calls,
    each with its own sampling locations and weights, captured once in a CUDA
    graph and replayed (no host work between layers)."""
    feats = make_feats(cams, CFG1_LEVELS, C, torch.float16, dev)
    ins = []
    for layer in range(layers):
        g = torch.Generator(device=dev).manual_seed(100 + layer)
        loc = torch.rand((1, Q, P, cams, 2), generator=g, device=dev)
        w = torch.softmax(torch.randn((1, Q, P * cams * 4, G), generator=g, device=dev), dim=2)
        ins.append((loc, w.reshape(1, Q, P, cams, 4, G).contiguous()))
    outs = [torch.empty((1, Q, C), device=dev) for _ in range(layers)]

    def frame():
        for (loc, w), o in zip(ins, outs):
            ops.deformable_aggregation(feats, None, None, loc, w, precision=precision, out=o)

    frame()  # workspace allocation outside the capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        frame()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            frame()
    torch.cuda.current_stream().wait_stream(s)
    med, best = time_fn(graph.replay, reps, flush=False)
    return {"config": "cfg3-frame", "path": f"{layers} x deformable_aggregation in one CUDA graph",
            "precision": precision, "dtype": "float16", "cams": cams, "layers": layers,
            "frame_us": med * 1e3, "best_us": best * 1e3, "per_layer_us": med * 1e3 / layers,
            "frames_per_s": 1e3 / med, "camera_streams_at_30fps": int(cams * (1e3 / med) / 30)}


def paint_case(reps, dev, cams=64, C=256, n_obj=40, n_occ=8):
    """Feature painting of a cfg3-shaped scene (64 ring cameras, 704x256
    images, strides 4-32, C=256) straight into the f16 table, device
    background: HBM-write bound (the table is the algorithmic byte count)."""
    K, R, T = ring(cams)
    camd = ops.Cameras(K, R, T, device=dev)
    rng = torch.Generator().manual_seed(9)
    ents = torch.cat([torch.rand((n_obj + n_occ, 2), generator=rng) * 8 - 4, torch.full((n_obj + n_occ, 1), 0.9),
                      torch.tensor([[0.6, 0.6, 1.8]]).repeat(n_obj + n_occ, 1),
                      torch.rand((n_obj + n_occ, 1), generator=rng) * 6.28 - 3.14], dim=1).double().numpy()
    sig = torch.nn.functional.normalize(torch.randn((n_obj, C), generator=rng, dtype=torch.float64), dim=1).numpy()
    wh = [[704, 256]] * cams
    strides = [4.0, 8.0, 16.0, 32.0]
    scene = ops.PaintScene(camd, wh, strides, C, ents, n_obj, sig)
    out = torch.empty((scene.rows, C), dtype=torch.float16, device=dev)
    fn = lambda: scene.run(sigma=0.01, seed=1, out=out)  # noqa: E731
    nbytes = out.numel() * 2
    med, best = time_fn(fn, reps, flush=False)
    gbs = nbytes / (med / 1e3) / 1e9
    return {"config": "paint-cfg3", "path": "paint (depth contest + signature + device N(0, sigma), f16 table)",
            "dtype": "float16", "cams": cams, "entities": n_obj + n_occ, "latency_us": med * 1e3,
            "best_us": best * 1e3, "table_bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peak()}


def assoc_case(reps, dev, n_q=900, n_d=900, D=256):
    """Association cost matrices for a 900-query bank vs 900 detections, D=256
    (the OAE embedding dimension at C=256), f64."""
    g = torch.Generator(device=dev).manual_seed(12)
    qc = torch.rand((n_q, 3), generator=g, device=dev, dtype=torch.float64) * 10 - 5
    dc = torch.rand((n_d, 3), generator=g, device=dev, dtype=torch.float64) * 10 - 5
    qe = torch.nn.functional.normalize(torch.randn((n_q, D), generator=g, device=dev, dtype=torch.float64), dim=1)
    de = torch.nn.functional.normalize(torch.randn((n_d, D), generator=g, device=dev, dtype=torch.float64), dim=1)
    fn = lambda: ops.association_cost(qc, dc, qe, de, 2.0, 1.0, 1.0, device=dev)  # noqa: E731
    med, best = time_fn(fn, reps, flush=False)
    return {"config": "assoc-900x900", "path": "association_cost (f64, numpy pairwise order)", "dtype": "float64",
            "n_q": n_q, "n_d": n_d, "dim": D, "latency_us": med * 1e3, "best_us": best * 1e3,
            "pairs_per_s": n_q * n_d / (med / 1e3)}


def fpyr_case(reps, dev, cams=6, C=256, frames=3):
    """FPYR container (cfg1 shape, 92 MB per frame) -> device table, per frame:
    one DMA from the page-locked mapping vs the pinned-staging path."""
    import os
    import tempfile

    from paper_2601_10819_b200 import features as F
    from paper_2601_10819_b200 import fpyr

    rng = np.random.default_rng(5)
    strides = [4.0, 8.0, 16.0, 32.0]
    frame = {c: F.FeaturePyramid(c, [F.FeatureGrid(stride=s, values=rng.uniform(-1, 1, (h, w, C)).astype(np.float32))
                                     for s, (h, w) in zip(strides, CFG1_LEVELS)]) for c in range(cams)}
    path = os.path.join(tempfile.mkdtemp(), "cfg1.fpyr")
    fpyr.write_pyramid_sequence(path, [frame] * frames)
    res = {}
    for pin in (True, False):
        with fpyr.FpyrReader(path, pin=pin) as rd:
            out = torch.empty((rd.header.rows, C), device=dev)
            rd.upload(0, device=dev, out=out)
            torch.cuda.synchronize()
            ts = []
            for i in range(reps):
                t0 = time.perf_counter()
                rd.upload(i % frames, device=dev, out=out)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            med = float(np.median(ts))
            res["pinned_mapping" if pin else "staged"] = {"ms": med * 1e3, "gbs": out.numel() * 4 / med / 1e9,
                                                          "registered": rd.registered}
    os.remove(path)
    return {"config": "fpyr-cfg1", "path": "FpyrReader.upload (frame -> channel-last device table)",
            "frame_bytes": int(out.numel() * 4), **res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cases = {
        "cfg1d": lambda: dense_case("cfg1 Sparse4D default (6 cams, G=8)", 6, CFG1_LEVELS, 256, 8, torch.float32,
                                    "fast", args.reps, dev),
        "cfg1d_exact": lambda: dense_case("cfg1 Sparse4D default, exact", 6, CFG1_LEVELS, 256, 8, torch.float32,
                                          "exact", max(3, args.reps // 4), dev),
        "cfg2d": lambda: dense_case("cfg2 warehouse 16x1080p (dense, G=8)", 16, CFG2_LEVELS, 256, 8,
                                    torch.float32, "fast", args.reps, dev),
        "cfg3": lambda: dense_case("cfg3 64 cams fp16 (per decoder layer)", 64, CFG1_LEVELS, 256, 8,
                                   torch.float16, "fast", args.reps, dev),
        "cfg3_h2": lambda: dense_case("cfg3 64 cams fp16, half2 accumulation", 64, CFG1_LEVELS, 256, 8,
                                      torch.float16, "fast_h2", args.reps, dev),
        "cfg3_exact": lambda: dense_case("cfg3 64 cams fp16, exact (bit-faithful f32 arithmetic)", 64, CFG1_LEVELS,
                                         256, 8, torch.float16, "exact", max(3, args.reps // 4), dev),
        "cfg4d": lambda: dense_case("cfg4 MSDA part: 32 cams bf16", 32, CFG1_LEVELS, 256, 8, torch.bfloat16, "fast",
                                    args.reps, dev),
        "cfg5": lambda: dense_case("cfg5 512 cams fp16 (1 GPU)", 512, CFG1_LEVELS, 256, 8, torch.float16, "fast",
                                   max(5, args.reps // 4), dev),
        "project": lambda: project_case(args.reps, dev),
        "frame": lambda: frame_case(max(5, args.reps // 2), dev),
        "frame_fast": lambda: frame_case(max(5, args.reps // 2), dev, precision="fast"),
        "paint": lambda: paint_case(args.reps, dev),
        "fpyr": lambda: fpyr_case(args.reps, dev),
        "assoc": lambda: assoc_case(args.reps, dev),
        "cfg4": lambda: oae_case(max(5, args.reps // 4), dev),
    }
    for name, fn in cases.items():
        if args.only and name not in args.only.split(","):
            continue
        try:
            print(json.dumps(fn()), flush=True)
        except Exception as e:  # keep going: one line per case
            print(json.dumps({"config": name, "error": repr(e)}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
