#!/usr/bin/env python
"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py gpurun_out/r1g profiles/r1 --config cfg2

Writes <dst>/ncu_<kernel>.md (key metrics of each full capture), the launch
list share table (<dst>/launches.md) and updates profiles/ncu_traffic.json
(dram read+write bytes per launch of the dominant kernel, consumed by
bench.py's roofline.traffic).
"""

from __future__ import annotations

import argparse
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {h: (row[i], units[i]) for i, h in enumerate(head) if i < len(row)}
        res.append(d)
    return res


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val.replace(",", "")) * scale.get(unit, 1)


def stalls(d):
    out = {}
    for k, (v, _) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                n = float(v.replace(",", ""))
            except ValueError:
                continue
            if n > 0:
                out[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = n
    return dict(sorted(out.items(), key=lambda kv: -kv[1])[:6])


def summarise_rep(rep: Path, dst: Path):
    lines = []
    traffic = None
    for d in raw(rep):
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## `{name}`\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        lines.append("\nTop stall reasons (pc samples): " +
                     ", ".join(f"{k} {int(v)}" for k, v in stalls(d).items()) + "\n")
        if "dram__bytes_read.sum" in d:
            traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
    out = dst / (f"ncu_{rep.stem}.md")
    out.write_text(f"# ncu --set full: {rep.name}\n\n" + "\n".join(lines) + "\n")
    return traffic


def summarise_launches(csv_path: Path, dst: Path):
    rows = [r for r in csv.reader(l for l in csv_path.read_text().splitlines() if not l.startswith("=="))]
    head = rows[0]
    ik, iv = head.index("Kernel Name"), head.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        tot[r[ik]] += float(r[iv].replace(",", ""))
        cnt[r[ik]] += 1
    # the timed step of bench.py (exact precision): the canonicaliser and the
    # exact gather (RAW = 0); everything else in the process (the fast-precision
    # leg, the e2e host-path fetch, torch helpers) is listed separately
    def in_step(k):
        if "plan_canon_kernel" in k:
            return True
        if "gather_pipe_kernel<" not in k:
            return False
        # template arguments <T, VEC, HALF, D, RAW, GW, DENSE, HACC>: the exact CSR gather has RAW = 0, GW = 1
        args = [a.strip() for a in k.split("gather_pipe_kernel<", 1)[1].split(">", 1)[0].split(",")]
        return len(args) >= 6 and args[4] == "0" and args[5] == "1" and (len(args) < 7 or args[6] == "0")

    def table(keys):
        total = sum(tot[k] for k in keys) or 1.0
        out = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k in sorted(keys, key=lambda k: -tot[k]):
            out.append(f"| `{k[:90]}` | {cnt[k]} | {tot[k] / cnt[k] / 1e3:.1f} | {tot[k] / total:.1%} |")
        return out

    step = [k for k in tot if in_step(k)]
    other = [k for k in tot if not in_step(k)]
    (dst / "launches.md").write_text(
        "# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n"
        "Cold-cache, serialised replays: compare shares, not absolutes.\n\n"
        "## The timed step (exact: plan_canon + gather)\n\n" + "\n".join(table(step)) +
        "\n\n## Other launches in the same bench process (fast-precision leg, e2e host path, torch)\n\n" +
        "\n".join(table(other)) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("dst")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--traffic-rep", default="prof_gather")
    args = ap.parse_args()
    src, dst = Path(args.src), Path(args.dst)
    dst.mkdir(parents=True, exist_ok=True)
    traffic = None
    for rep in sorted(src.glob("*.ncu-rep")):
        t = summarise_rep(rep, dst)
        if rep.stem == args.traffic_rep:
            traffic = t
    if (src / "launches.csv").exists():
        summarise_launches(src / "launches.csv", dst)
    for f in ("bench.json", "paths.jsonl"):
        if (src / f).exists():
            (dst / f).write_text((src / f).read_text())
    if traffic is not None:
        tj = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
        data = json.loads(tj.read_text()) if tj.exists() else {}
        data[args.config] = traffic
        tj.write_text(json.dumps(data, indent=1) + "\n")
    print(f"summaries in {dst}", file=sys.stderr)


if __name__ == "__main__":
    main()
