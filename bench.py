#!/usr/bin/env python
"""MSDA forward benchmark on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One step = one MSDA forward call over one batch (one scene) of the named
configuration.  Default workload = BASELINE configs[1] ("cfg2"): the
outside-in warehouse scene, 16 static cameras, 4 levels of 1080p-derived
features (270x480 .. 33x60, the reference bench generator's floor halving),
900 anchors x 13 keypoints per level per camera, C=256, fp32, exact
(bit-faithful) CSR path — inputs byte-identical to the reference's own
``generate_workload`` (seed = rank; rank 0 is the reference's seed 0).

Multi-GPU (torchrun): stream-sharded — every rank owns an independent scene
(no data-path collective); ``value`` = all ranks' camera-frames / max-rank
time.  ``--gpus N`` without torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU; it refuses to fold ranks
onto fewer GPUs unless ``BENCH_SHARE_GPU=1``, a smoke-test mode that is never
a measurement).  ``--impl reference`` times the reference's own CPU
implementation (``mvtrack3d.features.msda_optimized`` FULL from
``baseline/_ref``, all host threads; the oracle port when that install is
absent) on rank 0 only.

At N = 1 the line also carries a ``sparse4d`` block: the north_star operator
``deformable_aggregation`` at cfg1 (f32, f16), cfg2 (dense), cfg4 (bf16) and
the paper headline cfg3 (64 fp16 cameras, one frame = 6 decoder layers in one
CUDA graph), each checked against the C oracle before it is timed (EXACT:
bytes; FAST: 1e-4; FAST_H2: 1e-2), timed cold (L2 flushed) and warm with
CUDA events inside its own clock-sampling window.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2601_10819_b200.workload import BenchWorkload, generate_workload  # noqa: E402

METRIC = "MSDA fwd camera-streams/sec per B200 (camera-frames/s)"
CONFIGS = {
    "cfg2": dict(
        desc="outside-in warehouse scene: 16 static cams, 4 levels 270x480/135x240/67x120/33x60 (1080p strides "
             "4-32, reference bench floor halving), 900 anchors, 13 keypoints, C=256, fp32, exact CSR plan",
        wl=dict(cameras=16, levels=4, channels=256, queries=900, points_per_query=13, level0_size=(270, 480))),
    "cfg1": dict(
        desc="Sparse4D default shape as a CSR plan: 6 cams, 4 levels 64x176..8x22, 900 anchors, 13 keypoints, "
             "C=256, fp32, exact",
        wl=dict(cameras=6, levels=4, channels=256, queries=900, points_per_query=13, level0_size=(64, 176))),
    "default": dict(
        desc="reference BenchWorkload defaults: 6 cams, 4 levels 64x64..8x8, C=256, 900 queries, 13 points",
        wl=dict()),
}
L2_BYTES = 126 * 1024 * 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(config)
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU is busy."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(gw):
    """unique touched feature cells x C x 4 + plan inputs + outputs."""
    wl = gw.workload
    shape = gw.spatial_shape.reshape(-1, 2)
    t = gw.camera_ids.astype(np.int64) * wl.levels + gw.levels
    H = shape[t, 0].astype(np.int64)
    W = shape[t, 1].astype(np.int64)
    x0 = np.floor(gw.us).astype(np.int64)
    y0 = np.floor(gw.vs).astype(np.int64)
    rows = []
    for dy in (0, 1):
        for dx in (0, 1):
            x, y = x0 + dx, y0 + dy
            ok = (x >= 0) & (x < W) & (y >= 0) & (y < H)
            rows.append((gw.tile_start[t] + y * W + x)[ok])
    gathered = int(sum(r.size for r in rows))  # in-grid corner rows the gather moves (L2 -> SM)
    touched = np.unique(np.concatenate(rows)).size
    s_n, q_n = gw.us.size, wl.queries
    feat_b = touched * wl.channels * 4
    in_b = s_n * 20 + (q_n + 1) * 8
    out_b = q_n * wl.channels * 4 + q_n
    return {"touched_cells": int(touched), "touched_frac": touched / gw.table.shape[0], "feature_bytes": feat_b,
            "input_bytes": in_b, "output_bytes": out_b, "total": feat_b + in_b + out_b,
            "gathered_corner_bytes": gathered * wl.channels * 4}


def pcie_h2d_ceiling(dev, nbytes=512 << 20, reps=3):
    """Pinned host -> device copy-engine bandwidth (GB/s) on this box, the e2e leg's ceiling."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = float("inf")
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    del h, d
    return nbytes / (best / 1e3) / 1e9


def l2_gather_ceiling():
    """The measured L2 -> SM random-row gather ceiling of this part (no-math
    cp.async ring over the same rows, tools/gather_ceiling.cu), from the
    committed profile; None when absent."""
    p = ROOT / "profiles" / "r1" / "gather_ceiling.txt"
    if not p.exists():
        return None
    best = None
    for line in p.read_text().splitlines():
        if line.startswith("pipe_") and "moved" in line:
            v = float(line.split("moved")[1].split("GB/s")[0])
            best = v if best is None else max(best, v)
    return best


def reference_features():
    """The UNMODIFIED reference's ``mvtrack3d.features`` from ``baseline/_ref``
    (pip install of /root/reference), or None when absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "mvtrack3d" / "features.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from mvtrack3d import features as rf
    except Exception as e:  # pragma: no cover - broken install
        log(f"baseline/_ref present but mvtrack3d does not import ({e}); timing the oracle port")
        return None
    return rf


def host_metadata():
    """The reference's _host_metadata() (bench.py:130-139) plus the CPU model (lscpu)."""
    import platform

    md = {"platform": platform.platform(), "machine": platform.machine(), "python": platform.python_version(),
          "numpy": np.__version__, "cpu_count": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    md["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        md["affinity_cores"] = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        pass
    return md


def _cpu_impl(gw, workers):
    """A callable running the reference CPU algorithm on the first nq queries
    of the workload: the real mvtrack3d msda_optimized(FULL) when installed
    (kind "reference"), else the oracle port msda_tiled (kind "port")."""
    wl = gw.workload
    rf = reference_features()
    if rf is not None:
        pyrs = []
        for c in range(wl.cameras):
            lv = []
            for m, (h, w) in enumerate(wl.level_dims()):
                st = int(gw.tile_start[c * wl.levels + m])
                lv.append(rf.FeatureGrid(stride=wl.strides()[m], values=gw.table[st:st + h * w].reshape(h, w, -1)))
            pyrs.append(rf.FeaturePyramid(c, lv))

        def run(nq):
            s = int(gw.offsets[nq])
            plan = rf.SamplePlan.__new__(rf.SamplePlan)
            plan._finalize(np.ascontiguousarray(gw.offsets[:nq + 1]), gw.camera_ids[:s], gw.levels[:s], gw.us[:s],
                           gw.vs[:s], gw.weights[:s])
            return rf.msda_optimized(pyrs, plan, rf.PrecisionMode.FULL, workers=workers)
        return run, "reference", "mvtrack3d.features.msda_optimized(FULL, workers=%d) from baseline/_ref" % workers
    from oracle import msda_oracle as mo

    def run(nq):
        s = int(gw.offsets[nq])
        return mo.msda_tiled(gw.table, gw.tiles, wl.levels, gw.offsets[:nq + 1], gw.camera_ids[:s], gw.levels[:s],
                             gw.us[:s], gw.vs[:s], gw.weights[:s], precision="full", workers=workers)
    return run, "port", "oracle.msda_oracle.msda_tiled (msda_optimized FULL restated, numpy, ThreadPool)"


def cpu_reference_time(gw, budget_s=15.0, reps=3, workers=None):
    """Time the reference CPU algorithm (all host threads) on a bounded query
    sample; returns per-full-call seconds."""
    workers = workers or os.cpu_count() or 1
    wl = gw.workload
    per_q = wl.cameras * wl.levels * wl.points_per_query
    impl, kind, algo = _cpu_impl(gw, workers)

    def run(nq):
        t0 = time.perf_counter()
        out, _ = impl(nq)
        return time.perf_counter() - t0, out

    # The tile-grouped algorithm has a per-(camera, level) cost that a query
    # subset does not shrink, so a subset would over-state the full-call time:
    # time the whole workload unless one call exceeds the per-rep budget.
    t_full, out = run(wl.queries)  # warm-up and size probe
    nq = wl.queries
    if t_full > budget_s / reps:
        nq = max(2 * workers, int(wl.queries * (budget_s / reps) / t_full))
    times = []
    for _ in range(reps):
        t, out = run(nq)
        times.append(t)
    mean = float(np.mean(times))
    return {"full_call_s": mean * wl.queries / nq, "sample_queries": nq, "per_q_samples": per_q,
            "workers": workers, "times_s": times, "out": out, "kind": kind, "algorithm": algo}


def csr_config(args, cfg, wl):
    """The ``config`` object both arms print (identical keys and values)."""
    return {"workload": args.config, "desc": cfg["desc"],
            **{k: (list(v) if isinstance(v, tuple) else v) for k, v in wl.to_dict().items()}}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    wl = BenchWorkload(**cfg["wl"])
    gw = generate_workload(wl)
    workers = os.cpu_count() or 1
    # full workload per step unless warmup+steps would exceed ~3 minutes
    r = cpu_reference_time(gw, budget_s=max(1.0, 180.0 / max(1, args.steps + args.warmup)), reps=1,
                           workers=workers)
    nq = r["sample_queries"]
    impl, kind, algo = _cpu_impl(gw, workers)
    for _ in range(args.warmup):
        impl(nq)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        impl(nq)
        times.append(time.perf_counter() - t0)
    t_full = float(np.mean(times)) * wl.queries / nq
    value = wl.cameras / t_full
    sample = (f"the full workload per step ({wl.num_samples} samples)" if nq == wl.queries else
              f"{nq} of {wl.queries} queries per step ({nq * wl.cameras * wl.levels * wl.points_per_query} "
              f"samples), extrapolated linearly to the full call")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "camera-frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generate_workload)",
        "config": csr_config(args, cfg, wl),
        "cpu_baseline": {"value": value, "unit": "camera-frames/s", "cores": workers, "kind": kind,
                         "sample": sample, "algorithm": algo, "host": host_metadata()},
        "e2e": {"value": value, "unit": "camera-frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def rank_device(local_rank):
    """cuda:local_rank; BENCH_SHARE_GPU=1 (multi-rank smoke test on a one-GPU box) folds every rank onto the
    visible GPUs and uses gloo, since NCCL refuses two ranks on one device.  Never set for a measurement."""
    import torch

    if os.environ.get("BENCH_SHARE_GPU") == "1":
        return torch.device("cuda", local_rank % torch.cuda.device_count()), "gloo"
    if local_rank >= torch.cuda.device_count():
        raise SystemExit(f"rank {local_rank}: only {torch.cuda.device_count()} visible GPU(s); one rank per GPU "
                         "(BENCH_SHARE_GPU=1 folds ranks for a smoke test, never for a measurement)")
    return torch.device("cuda", local_rank), "nccl"


def run_ours(args, cfg, rank, local_rank, world):
    import torch
    import torch.distributed as dist

    from paper_2601_10819_b200 import features as F
    from paper_2601_10819_b200 import ops

    dev, backend = rank_device(local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group(backend, device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    wl = BenchWorkload(**{**cfg["wl"], "seed": rank})
    t0 = time.time()
    host_table = torch.empty((wl.num_rows, wl.channels), dtype=torch.float32, pin_memory=True)
    gw = generate_workload(wl, table_out=host_table.numpy())
    log(f"[rank {rank}] workload {args.config}: {wl.num_rows} rows x {wl.channels} ch "
        f"({host_table.numel() * 4 / 1e9:.2f} GB), {wl.num_samples} samples, generated in {time.time() - t0:.1f}s")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    feats = ops.DeviceFeatures(host_table.to(dev), t(gw.spatial_shape),
                               t(gw.tile_start.reshape(wl.cameras, wl.levels)))
    plan_d = [t(gw.offsets), t(gw.camera_ids), t(gw.levels), t(gw.us), t(gw.vs), t(gw.weights)]
    out = torch.empty((wl.queries, wl.channels), dtype=torch.float32, device=dev)
    empty = torch.empty((wl.queries,), dtype=torch.uint8, device=dev)
    table_bytes = host_table.numel() * 4
    flush = table_bytes < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    # correctness gate (raises on any device status) before timing
    ops.msda_csr(feats, *plan_d, out=out, empty=empty, check=True)

    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, args.warmup)):
        ops.msda_csr(feats, *plan_d, out=out, empty=empty, check=False)
    torch.cuda.synchronize(dev)

    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    smi_index = vis.split(",")[dev.index] if vis else str(dev.index)
    clocks = ClockSampler(smi_index)
    clocks.start()
    time.sleep(0.2)
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    # the step (status reset, canonicaliser, programmatically launched gather)
    # captured once in a CUDA graph and replayed: same kernels and bytes as the
    # eager call (tests/test_gpu_csr.py), without Python launch latency in the
    # first timed step
    step = lambda: ops.msda_csr(feats, *plan_d, out=out, empty=empty, check=False)  # noqa: E731
    graph = None
    try:
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            step()
        graph.replay()
        torch.cuda.synchronize(dev)
        ref_out = out.clone()
        step()
        torch.cuda.synchronize(dev)
        if not torch.equal(ref_out, out):
            raise RuntimeError("graph replay differs from the eager call")
        run_step = graph.replay
    except Exception as e:  # capture unsupported here: time the eager call
        log(f"[rank {rank}] CUDA graph capture unavailable ({e}); timing eager calls")
        graph, run_step = None, step
    barrier()
    torch.cuda.synchronize(dev)
    for k in range(K):  # the timed steps: one msda_csr call each (plan, then the gather launched programmatically)
        if flush:
            scratch.zero_()
        ev[k][0].record(stream)
        run_step()
        ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    # the two stages timed apart (events between them) for stage_us and the gather's roofline
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    for k in range(K):
        if flush:
            scratch.zero_()
        sev[k][0].record(stream)
        ops.msda_csr(feats, *plan_d, out=out, empty=empty, check=False, stages=1)
        sev[k][1].record(stream)
        ops.msda_csr(feats, *plan_d, out=out, empty=empty, check=False, stages=2)
        sev[k][2].record(stream)
    torch.cuda.synchronize(dev)
    # informational: FAST precision on the same plan (no canonicalisation; any
    # order, fused products) — one launch per call
    out_fast = torch.empty_like(out)
    ops.msda_csr(feats, *plan_d, out=out_fast, empty=empty, precision="fast", check=True)
    fev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    for k in range(K):
        if flush:
            scratch.zero_()
        fev[k][0].record(stream)
        ops.msda_csr(feats, *plan_d, out=out_fast, empty=empty, precision="fast", check=False)
        fev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    fast_ms = float(np.mean([fev[k][0].elapsed_time(fev[k][1]) for k in range(K)]))
    fast_err = float((out_fast - out).abs().max() / out.abs().max())
    # keep the GPU busy a little longer so the clock sampler sees load
    t_end = time.time() + 0.5
    while time.time() < t_end:
        ops.msda_csr(feats, *plan_d, out=out, empty=empty, check=False)
        torch.cuda.synchronize(dev)
    clk = clocks.stop()
    step_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(K)]
    plan_ms = [sev[k][0].elapsed_time(sev[k][1]) for k in range(K)]
    gather_ms = [sev[k][1].elapsed_time(sev[k][2]) for k in range(K)]
    total_ms = float(np.sum(step_ms))
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / K
    value = world * wl.cameras * K / (total_ms / 1e3)

    # ---- end to end through the reference-facing API (host buffers) ----
    pyrs = []
    for c in range(wl.cameras):
        lv = []
        for m, (h, w) in enumerate(wl.level_dims()):
            st = int(gw.tile_start[c * wl.levels + m])
            lv.append(F.FeatureGrid(stride=wl.strides()[m], values=gw.table[st:st + h * w].reshape(h, w, -1)))
        pyrs.append(F.FeaturePyramid(c, lv))
    # the step's inputs live in pinned host memory (features above, plan here)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    plan_h = F.SamplePlan.from_csr(*(pin(a) for a in (gw.offsets, gw.camera_ids, gw.levels, gw.us, gw.vs,
                                                        gw.weights)))
    e2e_k = max(1, min(K, args.e2e_steps))
    e2e_times = []
    for i in range(args.warmup + e2e_k):
        barrier()
        t1 = time.perf_counter()
        out_h, _ = F.msda_optimized(pyrs, plan_h, device=dev.index)
        dt = time.perf_counter() - t1
        if i >= args.warmup:
            e2e_times.append(dt)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    h2d = F.last_h2d_bytes(dev.index)  # whole grids copied + corner rows fetched from the sparse ones
    pcie = pcie_h2d_ceiling(dev)
    d2h = wl.queries * wl.channels * 4 + wl.queries
    same = out_h.tobytes() == out.cpu().numpy().tobytes()

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    ab = algorithmic_bytes(gw)
    peak, peak_src = measured_peak_hbm()
    g_ms = float(np.mean(gather_ms))
    achieved = ab["total"] / (g_ms / 1e3) / 1e9
    call_gbs = ab["total"] / (ms_per_step / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "camera-frames/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generate_workload bytes, seed=rank)",
        "config": csr_config(args, cfg, wl),
        "precision": "exact (bit-identical)",
        "parallelism": f"stream-sharded x{world} (independent scenes, no collective)",
        "l2": ("flushed between steps (2x L2 write)" if flush else
               f"inputs larger than L2 ({table_bytes / 1e9:.2f} GB table), no flush"),
        "latency_us": ms_per_step * 1e3,
        "stage_us": {"plan_canon": float(np.mean(plan_ms)) * 1e3, "gather_exact": g_ms * 1e3,
                     "note": "stages timed apart (events between them); the step is one call"},
        "streams_at_30fps_6layers": int(world * wl.cameras / (30 * 6 * ms_per_step / 1e3)),
        "call_gbs": call_gbs,
        "roofline": {"bound": "hbm", "kernel": "gather_pipe_kernel<float,4> (exact gather)", "achieved": achieved,
                     "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                     "peak_source": peak_src, "algorithmic_bytes": ab,
                     "secondary": {
                         "bound": "l2_gather",
                         "note": "the corner gathers (4 rows per sample, in-grid) cross L2 -> SM; DRAM sees each "
                                 "touched row about once",
                         "bytes": ab["gathered_corner_bytes"],
                         "achieved": ab["gathered_corner_bytes"] / (g_ms / 1e3) / 1e9,
                         "ceiling": l2_gather_ceiling(),
                         "ceiling_source": "measured: tools/gather_ceiling.cu no-math cp.async ring on the same rows "
                                           "(profiles/r1/gather_ceiling.txt)",
                         "unit": "GB/s"}},
        "e2e": {"value": world * wl.cameras / e2e_s, "unit": "camera-frames/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
                "api": "paper_2601_10819_b200.features.msda_optimized -> C-ABI msda_csr_host (pinned host buffers)",
                "transfer": "grids copied whole, except grids with more cells than 2 x the mean samples per grid "
                            "(levels 0-1 here): only their touched corner rows cross PCIe, fetched once each by the "
                            "device from the pinned buffer",
                "table_bytes": int(table_bytes),
                "bitwise_equal_to_device_path": same,
                "pcie": {"achieved_h2d_gbs": h2d / e2e_s / 1e9, "memcpy_h2d_gbs": pcie,
                         "frac": h2d / e2e_s / 1e9 / pcie,
                         "note": "memcpy_h2d_gbs = pinned 512 MiB cudaMemcpy H2D measured in this run (best of 3); "
                                 "device-warp zero-copy reads of 1 KB rows reach 0.93 of it "
                                 "(profiles/r1/pcie_ceiling.txt)"}},
        "fast_precision": {"ms_per_step": fast_ms, "value": world * wl.cameras / (fast_ms / 1e3),
                           "max_rel_err_vs_exact": fast_err,
                           "note": "precision='fast' on the same plan: one gather launch, no canonicalisation; "
                                   "informational (the headline is the bit-exact path)"},
        "gpu_launches": 2 * K,
        "step_mode": "CUDA graph replay of one msda_csr call" if graph is not None else "eager msda_csr call",
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu:
        r = cpu_reference_time(gw)
        nq = r["sample_queries"]
        parity = r["out"].tobytes() == out.cpu().numpy()[:nq].tobytes()
        line["cpu_baseline"] = {
            "value": wl.cameras / r["full_call_s"], "unit": "camera-frames/s", "cores": r["workers"],
            "kind": r["kind"],
            "sample": (f"full workload ({wl.num_samples} samples) x3 reps after 1 warm-up" if nq == wl.queries
                       else f"{nq} of {wl.queries} queries x3 reps (1 warm-up), extrapolated linearly"),
            "algorithm": r["algorithm"], "host": host_metadata(),
            "gpu_bitwise_equal_on_sample": bool(parity)}
        # SURVEY §8(d) also asks for the single-thread figure (msda_optimized, workers=1): one bounded rep
        r1 = cpu_reference_time(gw, budget_s=12.0, reps=1, workers=1)
        line["cpu_baseline"]["single_thread"] = {
            "value": wl.cameras / r1["full_call_s"], "unit": "camera-frames/s", "cores": 1, "kind": r1["kind"],
            "sample": (f"full workload x1 rep after 1 warm-up" if r1["sample_queries"] == wl.queries
                       else f"{r1['sample_queries']} of {wl.queries} queries x1 rep, extrapolated linearly")}
    if world == 1 and not args.no_sparse4d:
        del feats, plan_d, host_table, gw, pyrs, plan_h
        torch.cuda.empty_cache()
        line["sparse4d"] = sparse4d_block(args, dev, smi_index)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


SPARSE4D_CASES = [
    # (key, BASELINE config, cams, levels, dtype, precisions timed; the first is the case's headline)
    ("cfg1_f32", "configs[0] Sparse4D default: 6 cams, 64x176..8x22, 900 anchors, 13 pts, C=256, G=8, fp32", 6,
     "CFG1_LEVELS", "float32", ["fast", "exact"]),
    ("cfg1_f16", "configs[0] shape, fp16 features (PAPER.md's H100 fp16 comparison)", 6, "CFG1_LEVELS", "float16",
     ["fast_h2", "fast"]),
    ("cfg2_dense_f32", "configs[1] shape as the Sparse4D dense operator: 16 cams, 1080p levels 270x480..34x60, fp32",
     16, "CFG2_LEVELS", "float32", ["fast"]),
    ("cfg4_bf16", "configs[3] MSDA part: 32 cams at the cfg1 shape, bf16", 32, "CFG1_LEVELS", "bfloat16",
     ["fast", "exact"]),
    ("cfg3_f16", "configs[2] paper headline, one decoder layer: 64 cams at the cfg1 shape, fp16", 64, "CFG1_LEVELS",
     "float16", ["fast_h2", "fast", "exact"]),
]


def _time_events(fn, reps, stream, flush_buf=None):
    """Per-call CUDA-event times (ms) on ``stream``; ``flush_buf`` (> L2) is
    rewritten before every call (cold) or not at all (warm, back to back)."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in ev:
        if flush_buf is not None:
            flush_buf.zero_()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)


def sparse4d_block(args, dev, smi_index):
    """deformable_aggregation (north_star's operator) at the BASELINE shapes,
    under this run's clock: oracle parity first, then cold / warm timing."""
    import torch

    from oracle import build as ob  # the parity checker (test infrastructure), never the thing timed
    from paper_2601_10819_b200 import ops
    from tools import sparse4d_cases as s4

    peak, peak_src = measured_peak_hbm()
    ceiling = l2_gather_ceiling()
    stream = torch.cuda.current_stream(dev)
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    reps = max(5, args.steps)
    Q, P, G, C, L = 900, 13, 8, 256, 4
    res = {"note": "deformable_aggregation(mc_ms_feat, spatial_shape, scale_start_index, sampling_location, weights),"
                   " normalize=False (softmaxed weights, as Sparse4D); synthetic inputs per SURVEY 8(d); every "
                   "case is checked against the C oracle (oracle/msda_oracle.c, pinned to the reference) on the "
                   "features the GPU reads before it is timed; cold = L2 flushed (2x L2 write) before every call, "
                   "warm = back-to-back calls (the decoder-layer situation: same table, new anchors)",
           "peak_gbs": peak, "peak_source": peak_src, "l2_gather_ceiling_gbs": ceiling, "reps": reps, "cases": {}}
    clocks = ClockSampler(smi_index)
    clocks.start()
    time.sleep(0.2)
    t_block = time.time()
    for key, desc, cams, lv_name, dt_name, precs in SPARSE4D_CASES:
        levels = getattr(s4, lv_name)
        dtype = getattr(torch, dt_name)
        esize = torch.finfo(dtype).bits // 8
        feats = s4.make_feats(cams, levels, C, dtype, dev, seed=cams)
        loc, w = s4.make_dense_inputs(1, Q, P, cams, L, G, dev, seed=100 + cams)
        out = torch.empty((1, Q, C), dtype=torch.float32, device=dev)
        ab = s4.algorithmic_bytes(feats, loc, w, esize)
        # ---- parity against the C oracle on the features the GPU reads ----
        t0 = time.time()
        table, tiles, shape = s4.host_view(feats)
        loc_h, w_h = loc.cpu().numpy(), w.cpu().numpy()
        ref = ob.msda_dense_groups_c(table, tiles, shape, loc_h, w_h, L, normalize=False)
        oracle_s = time.time() - t0
        cpu_ref = None if getattr(args, "no_cpu", False) else _cpu_ref_dense(table, tiles, shape, loc_h, w_h, ref)
        del table
        scale = float(np.abs(ref).max())
        case = {"desc": desc, "cams": cams, "dtype": dt_name, "queries": Q, "points": P, "groups": G, "channels": C,
                "levels": [list(x) for x in levels], "algorithmic_bytes": ab,
                "l2": "flushed per call" if feats.table.numel() * esize < 2 * L2_BYTES else "table larger than L2",
                "oracle_s": oracle_s, "paths": {}}
        if cpu_ref is not None:
            case["cpu_reference"] = cpu_ref
        n_fine = s4.staged_fine_levels(levels, dtype)
        for prec in precs:
            fn = (lambda p=prec: ops.deformable_aggregation(feats, None, None, loc, w, precision=p, out=out))  # noqa
            # bytes that cross L2 -> SM as corner gathers: every level, or only
            # the fine ones when the coarse levels come from TMA-staged smem
            staged = n_fine is not None and prec != "exact"
            l2_bytes = (sum(ab["gathered_corner_bytes_per_level"][:n_fine]) if staged
                        else ab["gathered_corner_bytes"])
            ops.deformable_aggregation(feats, None, None, loc, w, precision=prec, out=out, check=True)
            got = out.cpu().numpy()
            err = float(np.abs(got - ref).max() / max(1e-12, scale))
            if prec == "exact":
                ok = got.tobytes() == ref.tobytes()
                parity = {"bitwise_equal_to_oracle": bool(ok)}
            else:
                tol = 1e-2 if prec == "fast_h2" else 1e-4
                ok = float(np.abs(got - ref).max() / (max(1.0, scale) if prec == "fast_h2" else scale)) <= tol
                parity = {"max_rel_err_vs_oracle": err, "tolerance": tol, "within_tolerance": bool(ok)}
            for _ in range(3):
                fn()
            cold = _time_events(fn, reps, stream, flush_buf)
            warm = _time_events(fn, reps, stream)
            med_c, med_w = cold[len(cold) // 2], warm[len(warm) // 2]
            achieved = ab["total"] / (med_c / 1e3) / 1e9
            case["paths"][prec] = {
                **parity, "latency_us": med_c * 1e3, "best_us": cold[0] * 1e3, "warm_us": med_w * 1e3,
                "vs_cpu_reference": (cpu_ref["full_call_s"] / (med_c / 1e3)) if cpu_ref else None,
                "camera_frames_per_s": cams / (med_c / 1e3),
                "streams_at_30fps_6layers": int(cams / (30 * 6 * med_c / 1e3)),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak},
                "path": ("levels 2-3 from TMA-staged shared memory (staged_coarse_kernel) + levels 0-1 by the "
                         "pipelined gather" if staged else
                         "fused one-pass exact gather" if prec == "exact" else "anchor-major pipelined gather"),
                "l2_gather": {"bytes": l2_bytes, "levels": f"0-{n_fine - 1}" if staged else "all",
                              "achieved_gbs": l2_bytes / (med_c / 1e3) / 1e9,
                              "frac_of_ceiling": (l2_bytes / (med_c / 1e3) / 1e9 / ceiling) if ceiling else None}}
        if key == "cfg3_f16":
            case["frame"] = _cfg3_frame(feats, dev, stream, reps, Q, P, G, C, L, cams)
        if key == "cfg4_bf16":
            case["full_path"] = _cfg4_full_path(feats, loc, w, out, dev, stream, flush_buf, reps, cams, Q, C,
                                                cpu=not getattr(args, "no_cpu", False))
        res["cases"][key] = case
        del feats, loc, w, out, ref
        torch.cuda.empty_cache()
    res["cases"]["cfg1_project_f32"] = _project_case(dev, stream, flush_buf, reps, peak)
    res["block_s"] = time.time() - t_block
    res["clocks"] = clocks.stop()
    return res


def _project_case(dev, stream, flush_buf, reps, peak, cams=6, Q=900, C=256, G=8, L=4):
    """north_star subsystem 2: keypoint generation + projection fused
    (msda_dense_project: f64 projection pre-pass, then the pipelined gather)
    at the cfg1 shape, against the plain operator on host-projected inputs'
    time; parity on 24 anchors vs the composed oracle (geometry.py:207-255 ->
    project_point -> pixel_to_cell -> msda_reference per group), 1e-4."""
    import torch

    from oracle import msda_oracle as mo
    from paper_2601_10819_b200 import ops
    from tools import sparse4d_cases as s4

    feats = s4.make_feats(cams, s4.CFG1_LEVELS, C, torch.float32, dev, seed=77)
    K, R, T = s4.ring(cams)
    camd = ops.Cameras(K, R, T, device=dev)
    anchors = s4.anchors_for(Q, dev).unsqueeze(0)
    offs = (torch.rand((6, 3), generator=torch.Generator().manual_seed(3)) * 2 - 1).to(dev)
    strides = torch.tensor([4.0, 8.0, 16.0, 32.0], device=dev)
    _, w = s4.make_dense_inputs(1, Q, 13, cams, L, G, dev, seed=78)
    out = torch.empty((1, Q, C), device=dev)
    fn = lambda: ops.msda_dense_project(feats, anchors, offs, camd, strides, w, dt=0.1, out=out)  # noqa: E731
    ops.msda_dense_project(feats, anchors, offs, camd, strides, w, dt=0.1, out=out, check=True)
    nq = 24
    table, tiles, _ = s4.host_view(feats)
    ref = mo.msda_project_groups(table, tiles, anchors[:, :nq].cpu().numpy(), offs.cpu().numpy(), K, R, T,
                                 [4.0, 8.0, 16.0, 32.0], w[:, :nq].cpu().numpy(), L, False, 0.1)
    err = float(np.abs(out[:, :nq].cpu().numpy() - ref).max() / max(1e-12, np.abs(ref).max()))
    for _ in range(3):
        fn()
    cold = _time_events(fn, reps, stream, flush_buf)
    warm = _time_events(fn, reps, stream)
    return {"desc": "cfg1 shape with keypoints (7 fixed + 6 learned) generated and projected (f64) from 900 anchors "
                    "through 6 ring cameras (704x256, f=300 px), fp32, FAST",
            "path": "msda_dense_project: projection pre-pass + pipelined gather",
            "latency_us": cold[len(cold) // 2] * 1e3, "warm_us": warm[len(warm) // 2] * 1e3,
            "max_rel_err_vs_oracle_24_anchors": err, "tolerance": 1e-4, "within_tolerance": err <= 1e-4}


def _cpu_ref_dense(table, tiles, shape, loc, w, oracle_out):
    """The reference CPU path for deformable_aggregation on this box (SURVEY
    8(c)/(d)): per channel group g, the UNMODIFIED mvtrack3d
    msda_optimized(FULL, normalize=False, all host threads) from
    baseline/_ref on the pyramids sliced to g's channels and the CSR plan of
    every (anchor, keypoint, camera, level) sample — cell = f32(f32(loc * W)
    - 0.5), weight w[..., g] — the composition the oracle restates.  One
    timed full call after a warm-up that builds the reference's packed-grid
    caches; its output is compared with the oracle's bytes, i.e. with the GPU
    EXACT path."""
    rf = reference_features()
    if rf is None:
        return None
    workers = os.cpu_count() or 1
    _, Q, P, cams, _ = loc.shape
    L, G, C = shape.shape[1], w.shape[-1], table.shape[1]
    cpg = C // G
    pyrs = [[rf.FeaturePyramid(c, [rf.FeatureGrid(stride=float(4 << m), values=np.ascontiguousarray(
        table[st:st + H * W, g * cpg:(g + 1) * cpg]).reshape(H, W, cpg))
        for m, (st, H, W) in enumerate(tiles[c * L:(c + 1) * L])]) for c in range(cams)] for g in range(G)]
    Hs, Ws = shape[:, :, 0].astype(np.float32), shape[:, :, 1].astype(np.float32)  # [cams, L]
    half = np.float32(0.5)

    def plans(nq):
        lx = loc[0, :nq, :, :, 0].astype(np.float32)[..., None]  # [nq, P, cams, 1]
        ly = loc[0, :nq, :, :, 1].astype(np.float32)[..., None]
        u = (lx * Ws[None, None]).astype(np.float32) - half  # features.py:20-24, two f32 roundings
        v = (ly * Hs[None, None]).astype(np.float32) - half
        cam_i = np.broadcast_to(np.arange(cams, dtype=np.int32)[None, None, :, None], u.shape)
        lvl_i = np.broadcast_to(np.arange(L, dtype=np.int32)[None, None, None, :], u.shape)
        offsets = np.arange(nq + 1, dtype=np.int64) * (P * cams * L)
        out = []
        for g in range(G):
            plan = rf.SamplePlan.__new__(rf.SamplePlan)
            plan._finalize(offsets, np.ascontiguousarray(cam_i).ravel(), np.ascontiguousarray(lvl_i).ravel(),
                           u.ravel(), v.ravel(), np.ascontiguousarray(w[0, :nq, ..., g], dtype=np.float32).ravel())
            out.append(plan)
        return out

    def run(nq):
        pl = plans(nq)
        t0 = time.perf_counter()
        res = [rf.msda_optimized(pyrs[g], pl[g], rf.PrecisionMode.FULL, normalize=False, workers=workers)[0]
               for g in range(G)]
        return time.perf_counter() - t0, np.concatenate(res, axis=1)

    run(min(Q, max(2 * workers, Q // 50)))  # warm-up: the reference's packed-pair caches of every grid
    t, got = run(Q)  # the full call (a query subset would over-state it: the per-tile costs dominate small subsets)
    return {"full_call_s": t, "camera_frames_per_s": cams / t, "cores": workers, "kind": "reference",
            "sample": f"the full call: {Q} anchors x {G} channel-group calls, 1 rep after a warm-up",
            "algorithm": f"mvtrack3d.features.msda_optimized(FULL, normalize=False, workers={workers}) per group "
                         "from baseline/_ref",
            "bitwise_equal_to_oracle": bool(got.tobytes() == oracle_out[0].tobytes())}


def _cpu_ref_oae(table, tiles, K, R, T, strides, anchors, offs, desc, vis, mem, emb, nq=16):
    """The reference's own occlusion-aware pooling on this host: for nq
    queries, generate_keypoints -> extract_view_feature on each of the 32
    cameras -> fuse_or_memory (oae.py:81-164; single-threaded Python as in
    the reference), extrapolated to all queries; its embeddings are compared
    with the GPU's."""
    ref = ROOT / "baseline" / "_ref"
    if reference_features() is None:
        return None
    from mvtrack3d import features as rf
    from mvtrack3d import geometry as rg
    from mvtrack3d import oae as ro

    cams = K.shape[0]
    L = len(strides)
    pyrs = [rf.FeaturePyramid(c, [rf.FeatureGrid(stride=float(s), values=table[st:st + H * W].reshape(H, W, -1))
                                  for s, (st, H, W) in zip(strides, tiles[c * L:(c + 1) * L])]) for c in range(cams)]
    cm = [rg.CameraModel(float(K[c, 0]), float(K[c, 1]), float(K[c, 2]), float(K[c, 3]), R[c], T[c], 704, 256)
          for c in range(cams)]
    err = 0.0
    t0 = time.perf_counter()
    for q in range(nq):
        st = rg.ObjectState3D(*(float(x) for x in anchors[q]))
        kp = rg.generate_keypoints(st, offs)
        memory = ro.Embedding.normalize(mem[q])
        query = ro.Query(track_id=q, anchor=st, memory=memory, descriptor=desc[q])
        pv = [ro.extract_view_feature(pyrs[c], cm[c], kp, query) for c in range(cams)]
        e = ro.fuse_or_memory(pv, list(vis[q]), memory)
        err = max(err, float(np.abs(e.values - emb[q]).max()))
    t = time.perf_counter() - t0
    Q = anchors.shape[0]
    return {"full_call_s": t * Q / nq, "queries_per_s": nq / t, "cores": 1, "kind": "reference",
            "sample": f"{nq} of {Q} queries x {cams} cameras, extrapolated linearly",
            "algorithm": "mvtrack3d.oae generate_keypoints + extract_view_feature + fuse_or_memory from "
                         f"{ref.relative_to(ROOT)}",
            "gpu_max_abs_err_on_sample": err}


def _cfg4_full_path(feats, loc, w, out, dev, stream, flush_buf, reps, cams, Q, C, cpu=True):
    """BASELINE configs[3]: the full aggregation path at 32 bf16 cameras —
    deformable_aggregation (FAST) over the feature table, then occlusion-aware
    ReID pooling on the same table (oae_pool: keypoints and f64 projection,
    level-mean f32 bilinear reads, softmax(desc . g / sqrt(D)), visibility-
    weighted fusion, L2 normalisation / memory fallback; oae.py:81-164).  OAE
    parity on 8 queries against the oracle (oae.py restated, f64) on the
    features the GPU reads, 1e-4 on the unit embedding; then cold / warm
    timing of the pooling alone and of the chained path."""
    import torch

    from oracle import msda_oracle as mo
    from paper_2601_10819_b200 import ops
    from tools import sparse4d_cases as s4

    K, R, T = s4.ring(cams)
    camd = ops.Cameras(K, R, T, device=dev)
    anchors = s4.anchors_for(Q, dev)
    offs = (torch.rand((6, 3), generator=torch.Generator().manual_seed(3)) * 2 - 1).to(dev)
    strides = [4.0, 8.0, 16.0, 32.0]
    strides_d = torch.tensor(strides, device=dev)
    g = torch.Generator(device=dev).manual_seed(4)
    desc = torch.randn((Q, C), generator=g, device=dev)
    vis = torch.rand((Q, cams), generator=g, device=dev)
    mem = torch.nn.functional.normalize(torch.randn((Q, C), generator=g, device=dev), dim=1)
    emb, occl = ops.oae_pool(feats, anchors, offs, camd, strides_d, desc, vis, mem, check=True)
    table, tiles, _ = s4.host_view(feats)
    nq, err, occ_ok = 8, 0.0, True
    an, of = anchors.cpu().double().numpy(), offs.cpu().double().numpy()
    de, vi, me = desc.cpu().double().numpy(), vis.cpu().numpy(), mem.cpu().double().numpy()
    e_host, o_host = emb[:nq].cpu().numpy(), occl[:nq].cpu().numpy()
    for q in range(nq):
        kps = mo.keypoints(an[q], of)
        views = [mo.extract_view(table, tiles, 4, c, strides, K[c], R[c], T[c], kps, de[q]) for c in range(cams)]
        ref, ref_occ = mo.fuse(views, vi[q], me[q])
        err = max(err, float(np.abs(e_host[q] - ref).max()))
        occ_ok &= bool(o_host[q]) == ref_occ
    cpu = _cpu_ref_oae(table, tiles, K, R, T, strides, an, of, de, vi, me, emb.cpu().numpy()) if cpu else None
    del table
    pool = lambda: ops.oae_pool(feats, anchors, offs, camd, strides_d, desc, vis, mem, check=False)  # noqa: E731

    def full():
        ops.deformable_aggregation(feats, None, None, loc, w, precision="fast", out=out)
        pool()

    res = {"desc": "MSDA (deformable_aggregation FAST, 900 anchors x 13 pts x 32 cams x 4 levels, G=8) then OAE "
                   "ReID pooling (900 queries: 7 fixed + 6 learned keypoints projected through 32 ring cameras, "
                   "4 levels, softmax over keypoints, visibility-weighted fusion) on the same bf16 table",
           "oae_max_abs_err_vs_oracle_8_queries": err, "oae_tolerance": 1e-4, "oae_occluded_flags_equal": occ_ok,
           "within_tolerance": bool(err <= 1e-4 and occ_ok)}
    if cpu is not None:
        res["cpu_reference_oae"] = cpu
    for name, fn in (("oae_pool", pool), ("msda_then_oae", full)):
        for _ in range(3):
            fn()
        cold = _time_events(fn, reps, stream, flush_buf)
        warm = _time_events(fn, reps, stream)
        res[name] = {"latency_us": cold[len(cold) // 2] * 1e3, "warm_us": warm[len(warm) // 2] * 1e3,
                     "vs_cpu_reference": (cpu["full_call_s"] / (cold[len(cold) // 2] / 1e3))
                     if (cpu and name == "oae_pool") else None,
                     "queries_per_s": Q / (cold[len(cold) // 2] / 1e3),
                     "camera_frames_per_s": cams / (cold[len(cold) // 2] / 1e3)}
    return res


def _cfg3_frame(feats, dev, stream, reps, Q, P, G, C, L, cams, layers=6):
    """The paper headline (BASELINE configs[2]): one frame of 64 fp16 camera
    streams = 6 decoder layers of deformable_aggregation, each with its own
    sampling locations and weights, captured once in a CUDA graph and
    replayed back to back (no host work between layers)."""
    import torch

    from paper_2601_10819_b200 import ops
    from tools import sparse4d_cases as s4

    ins = [s4.make_dense_inputs(1, Q, P, cams, L, G, dev, seed=200 + k) for k in range(layers)]
    outs = [torch.empty((1, Q, C), dtype=torch.float32, device=dev) for _ in range(layers)]
    frame = {}
    for prec in ("fast_h2", "fast"):
        def run(p=prec):
            for (loc, w), o in zip(ins, outs):
                ops.deformable_aggregation(feats, None, None, loc, w, precision=p, out=o)
        run()  # workspace allocation outside the capture
        torch.cuda.synchronize()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            run()
        graph.replay()
        torch.cuda.synchronize()
        t = _time_events(graph.replay, reps, stream)
        med = t[len(t) // 2]
        frame[prec] = {"frame_us": med * 1e3, "per_layer_us": med * 1e3 / layers, "frames_per_s": 1e3 / med,
                       "camera_streams_at_30fps": int(cams * (1e3 / med) / 30), "layers": layers}
        del graph
    return frame


DENSE_CONFIGS = {
    # cfg5 (BASELINE configs[4]): 512 cameras of the cfg1 per-camera shape, fp16, Sparse4D dense FAST path
    "cfg5-stream": dict(cams=512, scene=32, shard="stream",
                        desc="512 cams as 16 scenes x 32 cams, fp16, dense FAST, scenes dealt round-robin to ranks, "
                             "each rank's scenes aggregated as one batched call"),
    "cfg5-camera-peer": dict(cams=512, scene=512, shard="camera", transport="peer",
                             desc="one 512-cam scene, fp16, dense FAST, cameras split across ranks, partials pushed "
                                  "into every rank's buffer over NVLink (CUDA IPC, peer.cu) instead of NCCL"),
    "cfg5-camera": dict(cams=512, scene=512, shard="camera",
                        desc="one 512-cam scene, fp16, dense FAST, cameras split across ranks + NCCL partial-sum "
                             "all-reduce of [Q, C]"),
}
CFG1_LEVELS = [(64, 176), (32, 88), (16, 44), (8, 22)]


def _nccl_debug_setup(rank):
    """Before the process group exists: NCCL INFO logging into a per-rank
    file, so the bench line can say which algorithms / NVLS NCCL set up."""
    path = f"/tmp/msda_nccl.{os.getpid()}.{rank}.log"
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,TUNING,NVLS,GRAPH")
    os.environ["NCCL_DEBUG_FILE"] = path
    return path


def _nccl_report(path):
    import torch

    rep = {"version": ".".join(map(str, torch.cuda.nccl.version())) if hasattr(torch.cuda, "nccl") else None,
           "env": {k: os.environ[k] for k in ("NCCL_ALGO", "NCCL_PROTO", "NCCL_NVLS_ENABLE") if k in os.environ}}
    try:
        lines = Path(path).read_text(errors="replace").splitlines()
    except OSError:
        return {**rep, "log": "absent"}
    nvls = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "NVLS" in ln or "nvls" in ln]
    algo = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "Algo" in ln or "algorithm" in ln.lower()]
    rep.update({"nvls_lines": nvls[:8], "algo_lines": algo[:8], "log_lines": len(lines)})
    return rep


def run_dense_scaling(args, cfg, rank, local_rank, world):
    """cfg5 sweep (strong scaling: 512 cameras in total whatever N is)."""
    import torch
    import torch.distributed as dist

    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.dist import CameraShardedAggregation, camera_range, shard_streams

    dev, backend = rank_device(local_rank)
    torch.cuda.set_device(dev)
    nccl_log = _nccl_debug_setup(rank) if (world > 1 and backend == "nccl") else None
    if world > 1:
        dist.init_process_group(backend, device_id=dev)
    Q, P, G, C, L = 900, 13, 8, 256, 4
    gen = torch.Generator(device=dev).manual_seed(rank)

    def scene_feats(n_cams):
        rows = n_cams * sum(h * w for h, w in CFG1_LEVELS)
        table = (torch.rand((1, rows, C), generator=gen, device=dev) * 2 - 1).half()
        shape = torch.tensor([[list(x) for x in CFG1_LEVELS]] * n_cams, dtype=torch.int32)
        start = torch.tensor([[c * rows // n_cams + sum(h * w for h, w in CFG1_LEVELS[:m]) for m in range(L)]
                              for c in range(n_cams)], dtype=torch.int64)
        return ops.DeviceFeatures(table, shape, start)

    def inputs(n_cams):
        loc = torch.rand((1, Q, P, n_cams, 2), generator=gen, device=dev)
        w = torch.softmax(torch.randn((1, Q, P * n_cams * L, G), generator=gen, device=dev), dim=2)
        return loc, w.reshape(1, Q, P, n_cams, L, G).contiguous()

    step_mode = "eager"
    agg = None
    if cfg["shard"] == "stream":
        # this rank's scenes as ONE batched call: the scenes share the camera
        # and level geometry, so their tables stack as batch items [S, R, C]
        # (one launch fills the GPU; 16 sequential per-scene calls measured
        # 4.40 ms vs the batch below)
        mine = shard_streams(cfg["cams"] // cfg["scene"], rank, world)
        scenes = [scene_feats(cfg["scene"]) for _ in mine]
        ins = [inputs(cfg["scene"]) for _ in mine]
        if scenes:
            feats = ops.DeviceFeatures(torch.cat([f.table for f in scenes], 0), scenes[0].spatial_shape,
                                       scenes[0].scale_start_index)
            loc = torch.cat([x[0] for x in ins], 0)
            w = torch.cat([x[1] for x in ins], 0)
            del scenes, ins

        def step():
            if mine:
                ops.deformable_aggregation(feats, None, None, loc, w, precision="fast")
    else:
        lo, hi = camera_range(cfg["cams"], rank, world)
        feats = scene_feats(hi - lo)
        loc, w = inputs(hi - lo)  # this rank's cameras of the scene's sampling plan
        agg = CameraShardedAggregation.for_device_features(cfg["cams"], feats, precision="fast",
                                                           transport=cfg.get("transport", "collective"))

        def step():
            agg(loc, w, local_inputs=True, check=False)
        if agg.transport == "collective":
            # partial kernels + NCCL all-reduce + normalisation as one CUDA graph
            try:
                graph, _ = agg.capture(loc, w, normalize=True, local_inputs=True)
                step, step_mode = graph.replay, "CUDA graph: partial + all-reduce + normalise"
            except Exception as e:  # e.g. a gloo group (BENCH_SHARE_GPU): no capture, eager calls
                log(f"[rank {rank}] capture unavailable ({type(e).__name__}: {e}); eager calls")
                step = lambda: agg(loc, w, normalize=True, local_inputs=True, check=False)  # noqa: E731
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step()
    b.record()
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / args.steps
    per_rank = [ms]
    if world > 1:
        t = torch.tensor([ms], device=dev)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        per_rank = [float(x.item()) for x in gathered]
        ms = max(per_rank)
    if rank == 0:
        line = {
            "metric": METRIC, "value": cfg["cams"] / (ms / 1e3), "unit": "camera-frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f16", "data": "synthetic (device RNG)",
            "config": {"workload": args.config, "desc": cfg["desc"], "queries": Q, "points": P, "groups": G,
                       "channels": C, "levels": CFG1_LEVELS},
            "per_rank_ms": per_rank, "step_mode": step_mode, "backend": backend,
            "streams_at_30fps_6layers": int(cfg["cams"] / (30 * 6 * ms / 1e3))}
        if nccl_log:
            line["nccl"] = _nccl_report(nccl_log)
        print(json.dumps(line), flush=True)
    if agg is not None:
        agg.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def launch_ranks(args):
    """``--gpus N`` without torchrun: re-run this script under
    ``torch.distributed.run`` with N ranks on this node (127.0.0.1), one per
    GPU.  Refuses (exit 2) when fewer than N GPUs are visible, unless
    BENCH_SHARE_GPU=1 (ranks folded onto the visible GPUs over gloo: a smoke
    test of the multi-rank path, never a measurement)."""
    import socket

    if os.environ.get("BENCH_PLUMBING") != "1":
        import torch

        n = torch.cuda.device_count()
        if n < args.gpus and os.environ.get("BENCH_SHARE_GPU") != "1":
            log(f"bench.py --gpus {args.gpus}: only {n} GPU(s) visible; one rank per GPU is required "
                "(BENCH_SHARE_GPU=1 folds ranks for a smoke test, not a measurement)")
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    log("launching: " + " ".join(cmd))
    return subprocess.call(cmd)


def run_plumbing(args, rank, world):
    """BENCH_PLUMBING=1 (CPU tests only): the multi-rank launch, barrier,
    max-over-ranks and JSON path of the bench over gloo with a trivial host
    step — no GPU, no measurement."""
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    import torch

    a = np.ones((256, 256), dtype=np.float32)
    for _ in range(args.warmup):
        a @ a
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a @ a
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "camera-frames/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(t.item()) / args.steps * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                          "data": "plumbing test (BENCH_PLUMBING=1): no GPU, no measurement",
                          "config": {"workload": args.config}}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS) + sorted(DENSE_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sparse4d", action="store_true", help="skip the sparse4d block")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, local_rank, world = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(launch_ranks(args))
    if args.impl == "ours" and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if os.environ.get("BENCH_PLUMBING") == "1":
        run_plumbing(args, rank, world)
        return
    if args.config in DENSE_CONFIGS:
        run_dense_scaling(args, DENSE_CONFIGS[args.config], rank, local_rank, world)
        return
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_ours(args, cfg, rank, local_rank, world)


if __name__ == "__main__":
    main()
