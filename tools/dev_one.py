#!/usr/bin/env python
"""Builder loop: one deformable_aggregation case (cams, dtype, precision)
called a few times, for ncu launch lists / captures."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2601_10819_b200 import ops  # noqa: E402
from tools import sparse4d_cases as s4  # noqa: E402

cams, dt, prec = int(sys.argv[1]), sys.argv[2], sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dev = torch.device("cuda", 0)
levels = s4.CFG2_LEVELS if cams == 16 else s4.CFG1_LEVELS
feats = s4.make_feats(cams, levels, 256, getattr(torch, dt), dev, seed=cams)
loc, w = s4.make_dense_inputs(1, 900, 13, cams, 4, 8, dev, seed=100 + cams)
out = torch.empty((1, 900, 256), device=dev)
for _ in range(reps):
    ops.deformable_aggregation(feats, None, None, loc, w, precision=prec, out=out)
torch.cuda.synchronize()
print("done")
