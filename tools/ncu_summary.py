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


def opcode_mix(rep: Path, top=16):
    """Executed SASS instructions per opcode (all kernels of the capture), from the source page."""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    mixes, cur = [], None
    for row in csv.reader(out.splitlines()):
        if len(row) >= 2 and row[0] == "Kernel Name":
            cur = [row[1], defaultdict(int), None]
            mixes.append(cur)
            continue
        if cur is None or not row:
            continue
        if row[0] == "Address":
            cur[2] = (row.index("Source"), row.index("Instructions Executed"))
            continue
        if cur[2] is None or len(row) <= cur[2][1]:
            continue
        try:
            n = int(row[cur[2][1]])
        except ValueError:
            continue
        t = row[cur[2][0]].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        cur[1][op.split(".")[0]] += n
    res = []
    for name, mix, _ in mixes:
        total = sum(mix.values()) or 1
        res.append((name, total, sorted(mix.items(), key=lambda kv: -kv[1])[:top]))
    return res


def summarise_rep(rep: Path, dst: Path):
    lines = []
    traffic = None
    mixes = opcode_mix(rep)  # same kernel order as the raw page
    for i, d in enumerate(raw(rep)):
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## `{name}`\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        lines.append("\nTop stall reasons (pc samples): " +
                     ", ".join(f"{k} {int(v)}" for k, v in stalls(d).items()) + "\n")
        mix = mixes[i] if i < len(mixes) else None
        if mix:
            lines.append(f"Executed SASS opcodes (top of {mix[1]:,}): " +
                         ", ".join(f"{op} {n / mix[1]:.1%}" for op, n in mix[2]) + "\n")
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
    for extra in sorted(src.glob("launches_*.csv")):  # other launch lists: plain per-kernel tables
        rows = [r for r in csv.reader(l for l in extra.read_text().splitlines() if not l.startswith("=="))]
        if not rows:
            continue
        ik, iv = rows[0].index("Kernel Name"), rows[0].index("Metric Value")
        tot, cnt = defaultdict(float), defaultdict(int)
        for r in rows[1:]:
            tot[r[ik]] += float(r[iv].replace(",", ""))
            cnt[r[ik]] += 1
        total = sum(tot.values()) or 1.0
        body = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k in sorted(tot, key=lambda k: -tot[k]):
            body.append(f"| `{k[:90]}` | {cnt[k]} | {tot[k] / cnt[k] / 1e3:.1f} | {tot[k] / total:.1%} |")
        (dst / f"{extra.stem}.md").write_text(f"# ncu launch list {extra.name} (gpu__time_duration.sum)\n\n" +
                                              "\n".join(body) + "\n")
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
