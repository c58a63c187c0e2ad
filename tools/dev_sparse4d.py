#!/usr/bin/env python
"""Builder loop: bench.py's sparse4d block alone (oracle parity + cold/warm
timing per case), printed compactly.  ``--only cfg3_f16,cfg1_f32`` narrows it."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--json", default="")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference legs")
    args = ap.parse_args()
    import torch

    if args.only:
        keep = set(args.only.split(","))
        bench.SPARSE4D_CASES[:] = [c for c in bench.SPARSE4D_CASES if c[0] in keep]
    args.no_sparse4d = False
    dev = torch.device("cuda", 0)
    res = bench.sparse4d_block(args, dev, "0")
    if args.json:
        Path(args.json).write_text(json.dumps(res))
    for key, c in res["cases"].items():
        if "paths" not in c:
            print(key, {k: v for k, v in c.items() if k not in ("desc",)})
            continue
        for p, v in c["paths"].items():
            par = "bits" if v.get("bitwise_equal_to_oracle") else (
                f"err {v['max_rel_err_vs_oracle']:.1e}" if "max_rel_err_vs_oracle" in v else "MISMATCH")
            ok = v.get("bitwise_equal_to_oracle", v.get("within_tolerance"))
            print(f"{key:16s} {p:8s} {v['latency_us']:8.1f} us cold {v['warm_us']:8.1f} warm  "
                  f"hbm {v['roofline']['frac']:.3f}  l2 {v['l2_gather']['frac_of_ceiling'] or 0:.2f}  {par} "
                  f"{'OK' if ok else 'FAIL'}")
        if "cpu_reference" in c:
            cr = c["cpu_reference"]
            print(f"{key:16s} cpu reference {cr['full_call_s'] * 1e3:.0f} ms ({cr['cores']} cores), bitwise "
                  f"{cr['bitwise_equal_to_oracle']}")
        if "full_path" in c:
            fp = c["full_path"]
            print(f"{key:16s} full path: oae {fp['oae_pool']['latency_us']:.1f} us cold, msda+oae "
                  f"{fp['msda_then_oae']['latency_us']:.1f} us cold, oae err {fp['oae_max_abs_err_vs_oracle_8_queries']:.1e} "
                  f"{'OK' if fp['within_tolerance'] else 'FAIL'}")
            if "cpu_reference_oae" in fp:
                co = fp["cpu_reference_oae"]
                print(f"{key:16s} cpu reference oae {co['full_call_s'] * 1e3:.0f} ms, err {co['gpu_max_abs_err_on_sample']:.1e}")
        if "frame" in c:
            for p, v in c["frame"].items():
                print(f"{key:16s} frame {p:8s} {v['frame_us']:8.1f} us  per layer {v['per_layer_us']:.1f}")
    print("clocks", res["clocks"])


if __name__ == "__main__":
    main()
