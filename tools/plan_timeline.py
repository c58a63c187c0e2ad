#!/usr/bin/env python
"""Builder tool: per-CTA globaltimer timeline of the exact CSR step (cfg2).

Needs a library built with ``MSDA_EXTRA_NVCC_FLAGS=-DMSDA_PLAN_TL`` (never
shipped).  Prints, relative to the first plan CTA's start, the distribution of
each plan phase end (loads, run table, ranks + records, sum, CTA end) and of
the gather warps' start / griddepcontrol.wait return / end, with the gather
warps per SM and each SM's last end (DESIGN §10 "Gather placement")."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2601_10819_b200 import _lib, ops  # noqa: E402
from paper_2601_10819_b200.workload import BenchWorkload, generate_workload  # noqa: E402

dev = torch.device("cuda", 0)
wl = BenchWorkload(**{**bench.CONFIGS["cfg2"]["wl"], "seed": 0})
host = torch.empty((wl.num_rows, wl.channels), dtype=torch.float32, pin_memory=True)
gw = generate_workload(wl, table_out=host.numpy())
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
feats = ops.DeviceFeatures(host.to(dev), t(gw.spatial_shape), t(gw.tile_start.reshape(wl.cameras, wl.levels)))
plan = [t(gw.offsets), t(gw.camera_ids), t(gw.levels), t(gw.us), t(gw.vs), t(gw.weights)]
out = torch.empty((wl.queries, wl.channels), dtype=torch.float32, device=dev)
empty = torch.empty((wl.queries,), dtype=torch.uint8, device=dev)
for _ in range(5):
    ops.msda_csr(feats, *plan, out=out, empty=empty, check=False)
torch.cuda.synchronize()
buf = np.zeros((8192, 8), dtype=np.uint64)
lib = _lib.lib()
rc = lib.msda_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
assert rc == 0, rc
nq = wl.queries
plan_t = buf[:nq, :6].astype(np.int64)
t0 = plan_t[:, 0].min()
rows = 2048 + np.nonzero(buf[2048:, 2])[0]
gat = buf[rows, :3].astype(np.int64)
pct = lambda x: " ".join(f"{np.percentile(x, p) / 1e3:7.2f}" for p in (0, 10, 50, 90, 100))  # noqa: E731
print("us rel. to first plan CTA start:   min     p10     p50     p90     max")
for k, name in enumerate(["plan start", "loads+keys", "run table", "ranks+records", "sum", "plan end"]):
    print(f"{name:16s} {pct(plan_t[:, k] - t0)}")
for k, name in enumerate(["gather start", "gather wait ret", "gather end"]):
    print(f"{name:16s} {pct(gat[:, k] - t0)}")
print("per-CTA phase durations (p50 us):",
      " ".join(f"{np.median(plan_t[:, k + 1] - plan_t[:, k]) / 1e3:.2f}" for k in range(5)))
sm = buf[rows, 3].astype(np.int64)
end = (gat[:, 2] - t0) / 1e3
cnt = np.bincount(sm, minlength=148)
print("gather warps per SM:", dict(zip(*np.unique(cnt, return_counts=True))))
for c in np.unique(cnt):
    sel = cnt[sm] == c
    if sel.any():
        print(f"  SMs with {c} warps: end p50 {np.median(end[sel]):.1f} max {end[sel].max():.1f} us")
sm_end = np.array([end[sm == i].max() if (sm == i).any() else 0 for i in range(148)])
print("per-SM last end (us) by smid, 16 per line:")
for i in range(0, 148, 16):
    print("  ", " ".join(f"{x:5.0f}" for x in sm_end[i:i + 16]))
order = np.argsort(end)
print("gather warps:", len(rows))
