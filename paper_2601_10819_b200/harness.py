"""The reference's MSDA benchmark harness, on the GPU path.

Mirrors ``mvtrack3d.bench.bench_msda`` / ``write_report`` (bench.py:142-194),
the ``bench_workload_v1`` schema (schemas/bench_workload_v1.schema.json,
fail-closed) and the ``bench-msda`` CLI subcommand (cli.py:229-247, 379-384,
exit codes of cli.py:404-422) so existing reports and tooling keep working:
same report keys (workload echo, host metadata, timer, input checksum,
reference/optimized mean/min/max/times, speedup, cameras_at_fps) plus a
``device`` block.  "reference" times the reference-semantics entry point
(``features.msda_reference``), "optimized" times ``features.msda_optimized``
at the requested precision; both are the GPU path through the C ABI with host
arrays in and out (wall clock around a synchronous call, the reference's own
methodology, bench.py:116-127).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import platform
import sys
import time
import traceback
from pathlib import Path

import numpy as np

from . import __version__
from .workload import BenchWorkload, generate_workload

_SCHEMA_FIELDS = {
    "schema_version": "const1", "cameras": ("int", 1), "levels": ("int", 1), "channels": ("int", 2),
    "queries": ("int", 1), "points_per_query": ("int", 1), "level0_size": "size2", "repetitions": ("int", 0),
    "seed": ("int", 0), "fps_targets": "fps",
}


class ConfigError(ValueError):
    """A configuration document failed validation (errors.py:300-301)."""


def validate_workload_doc(doc) -> None:
    """Fail-closed check of a ``bench_workload_v1`` document."""
    if not isinstance(doc, dict):
        raise ConfigError("bench_workload_v1: document must be an object")
    unknown = sorted(set(doc) - set(_SCHEMA_FIELDS))
    if unknown:
        raise ConfigError(f"bench_workload_v1: unknown field(s) {unknown}")
    if doc.get("schema_version") != 1:
        raise ConfigError("bench_workload_v1: schema_version must be 1")
    for key, rule in _SCHEMA_FIELDS.items():
        if key not in doc or key == "schema_version":
            continue
        val = doc[key]
        if isinstance(rule, tuple):
            if isinstance(val, bool) or not isinstance(val, int) or val < rule[1]:
                raise ConfigError(f"bench_workload_v1: {key} must be an integer >= {rule[1]}")
        elif rule == "size2":
            if (not isinstance(val, list) or len(val) != 2 or
                    any(isinstance(x, bool) or not isinstance(x, int) or x < 1 for x in val)):
                raise ConfigError("bench_workload_v1: level0_size must be [height, width], integers >= 1")
        elif rule == "fps":
            if (not isinstance(val, list) or
                    any(isinstance(x, bool) or not isinstance(x, (int, float)) or not x > 0 for x in val)):
                raise ConfigError("bench_workload_v1: fps_targets must be positive numbers")


def workload_from_dict(doc) -> BenchWorkload:
    """``BenchWorkload.from_dict`` (bench.py:40-48)."""
    validate_workload_doc(doc)
    kw = {k: v for k, v in doc.items() if k != "schema_version"}
    if "level0_size" in kw:
        kw["level0_size"] = tuple(kw["level0_size"])
    if "fps_targets" in kw:
        kw["fps_targets"] = tuple(kw["fps_targets"])
    return BenchWorkload(**kw)


def _time_path(fn, repetitions: int) -> dict:
    times = []
    for _ in range(repetitions):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return {"mean_s": float(np.mean(times)), "min_s": float(np.min(times)), "max_s": float(np.max(times)),
            "times_s": [float(t) for t in times]}


def _host_metadata() -> dict:
    import os

    return {"platform": platform.platform(), "machine": platform.machine(), "python": platform.python_version(),
            "numpy": np.__version__, "cpu_count": os.cpu_count()}


def _pyramids(gw):
    from .features import FeatureGrid, FeaturePyramid

    wl = gw.workload
    out = []
    for c in range(wl.cameras):
        lv = []
        for m, (h, w) in enumerate(wl.level_dims()):
            st = int(gw.tile_start[c * wl.levels + m])
            lv.append(FeatureGrid(stride=wl.strides()[m], values=gw.table[st:st + h * w].reshape(h, w, -1)))
        out.append(FeaturePyramid(c, lv))
    return out


def bench_msda(workload: BenchWorkload, mode="full", workers: int = 1, device: int = 0) -> dict:
    """Time both entry points on the workload (bench.py:142-188 semantics)."""
    from . import features as F

    mode_e = F.PrecisionMode(mode) if not isinstance(mode, F.PrecisionMode) else mode
    report = {
        "schema_version": 1,
        "tool_version": __version__,
        "workload": workload.to_dict(),
        "mode": mode_e.value,
        "workers": int(workers),
        "host": _host_metadata(),
        "timer": {"name": "perf_counter", "resolution_s": time.get_clock_info("perf_counter").resolution},
    }
    if workload.repetitions == 0:
        report["measured"] = False
        return report
    gw = generate_workload(workload)
    report["input_checksum"] = gw.checksum
    pyrs = _pyramids(gw)
    plan = F.SamplePlan.from_csr(gw.offsets, gw.camera_ids, gw.levels, gw.us, gw.vs, gw.weights)
    F.msda_reference(pyrs, plan, device=device)
    F.msda_optimized(pyrs, plan, mode_e, workers=workers, device=device)
    ref = _time_path(lambda: F.msda_reference(pyrs, plan, device=device), workload.repetitions)
    opt = _time_path(lambda: F.msda_optimized(pyrs, plan, mode_e, workers=workers, device=device),
                     workload.repetitions)
    report["measured"] = True
    report["reference"] = ref
    report["optimized"] = opt
    report["speedup"] = ref["mean_s"] / opt["mean_s"] if opt["mean_s"] > 0 else float("inf")
    cams = {}
    for fps in workload.fps_targets:
        pr, po = ref["mean_s"] / workload.cameras, opt["mean_s"] / workload.cameras
        cams[f"{fps:g}"] = {"reference": int(1.0 / (fps * pr)) if pr > 0 else 0,
                            "optimized": int(1.0 / (fps * po)) if po > 0 else 0}
    report["cameras_at_fps"] = cams
    try:
        import torch

        report["device"] = {"name": torch.cuda.get_device_name(device), "index": device,
                            "path": "C-ABI msda_csr_host (host arrays in/out, copies included)"}
    except Exception:  # noqa: BLE001 - metadata only
        report["device"] = {"index": device}
    return report


def write_report(report: dict, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(report, fh, indent=2, sort_keys=True)
        fh.write("\n")


def _sha256_file(path) -> str:
    return "sha256:" + hashlib.sha256(Path(path).read_bytes()).hexdigest()


def _load_json(path):
    text = Path(path).read_text(encoding="utf-8")
    try:
        return json.loads(text)
    except json.JSONDecodeError as exc:
        raise ConfigError(f"{path}: invalid JSON at line {exc.lineno} column {exc.colno}: {exc.msg}") from exc


def _cmd_bench_msda(args) -> int:
    out_dir = Path(args.out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    t0 = time.perf_counter()
    inputs = {}
    doc = {"schema_version": 1}
    if args.config:
        doc = _load_json(args.config)
        inputs[str(args.config)] = _sha256_file(args.config)
    if args.seed_override is not None:
        doc = dict(doc)
        doc["seed"] = args.seed_override
    workload = workload_from_dict(doc)
    ts = time.perf_counter()
    report = bench_msda(workload, mode=args.mode, workers=args.workers, device=args.device)
    t_bench = time.perf_counter() - ts
    out = Path(args.out) if args.out else out_dir / "bench.json"
    if out.parent != Path("."):
        out.parent.mkdir(parents=True, exist_ok=True)
    write_report(report, out)
    manifest = {"tool": "paper_2601_10819_b200", "tool_version": __version__, "subcommand": "bench-msda",
                "config": {"workload": workload.to_dict()}, "inputs": inputs,
                "outputs": [str(out) if args.out else "bench.json"], "workers": args.workers,
                "seed_override": args.seed_override,
                "timings_s": {"bench": round(t_bench, 6), "total": round(time.perf_counter() - t0, 6)}}
    write_report(manifest, out_dir / "manifest.json")
    if report.get("measured", False):
        print(f"reference {report['reference']['mean_s']:.6f}s  optimized {report['optimized']['mean_s']:.6f}s  "
              f"speedup {report['speedup']:.2f}x")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2601_10819_b200")
    sub = p.add_subparsers(dest="cmd")
    b = sub.add_parser("bench-msda", help="time the reference-semantics vs optimized aggregation on the GPU")
    b.add_argument("--config", default=None, help="workload JSON (schema bench_workload_v1); defaults apply")
    b.add_argument("--mode", choices=("full", "half"), default="full", help="optimized-path precision")
    b.add_argument("--out", default=None, help="report JSON path (default: <out-dir>/bench.json)")
    b.add_argument("--out-dir", default=".")
    b.add_argument("--workers", type=int, default=1, help="accepted for compatibility; the GPU ignores it")
    b.add_argument("--seed-override", type=int, default=None)
    b.add_argument("--device", type=int, default=0)
    b.set_defaults(fn=_cmd_bench_msda)
    return p


def main(argv=None) -> int:
    """Exit 0 ok, 1 validation / IO error, 2 anything else (cli.py:404-422)."""
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else 1
    if getattr(args, "fn", None) is None:
        parser.print_usage(sys.stderr)
        return 1
    try:
        return args.fn(args)
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except Exception:  # noqa: BLE001
        traceback.print_exc()
        return 2
