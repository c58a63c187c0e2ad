"""Multi-rank bench modes and the graph-captured camera-sharded call on the
one-GPU box: ranks are folded onto the visible GPU with BENCH_SHARE_GPU=1
(gloo), which exercises bench.py's launcher, the stream-sharded and
camera-sharded drivers and max-over-ranks timing — never a measurement."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import helpers
from oracle import msda_oracle as mo

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _bench(*args, timeout=900):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["BENCH_SHARE_GPU"] = "1"
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config", ["cfg5-stream", "cfg5-camera"])
def test_bench_two_ranks_folded(cuda_dev, config):
    d = _bench("--gpus", "2", "--config", config, "--steps", "2", "--warmup", "3")
    assert d["n_gpus"] == 2 and d["value"] > 0 and len(d["per_rank_ms"]) == 2
    assert d["ms_per_step"] == max(d["per_rank_ms"])


def test_bench_csr_two_ranks_folded(cuda_dev):
    """The headline CSR mode stream-sharded over 2 ranks (each its own scene, seed = rank)."""
    d = _bench("--gpus", "2", "--config", "cfg1", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-sparse4d",
               "--e2e-steps", "1")
    assert d["n_gpus"] == 2 and d["value"] > 0 and "stream-sharded x2" in d["parallelism"]


def test_camera_sharded_capture_matches_eager(cuda_dev):
    """One rank: CameraShardedAggregation.capture (partial kernels +
    normalisation in one CUDA graph over static inputs) equals the eager call
    and the oracle; replays pick up new inputs written in place."""
    import torch

    from paper_2601_10819_b200 import ops
    from paper_2601_10819_b200.dist import CameraShardedAggregation

    rng = np.random.default_rng(21)
    grids, shape, loc, wts = helpers.make_dense(rng, bs=1, n_q=30, n_p=13, cams=5, n_levels=4, groups=8,
                                                channels=256, size_lo=8, size_hi=30)
    table, tiles = mo.pack_grids(grids, 5, 4)
    start = np.array([t[0] for t in tiles], dtype=np.int64).reshape(5, 4)
    feats = ops.DeviceFeatures(torch.from_numpy(table).to(cuda_dev), torch.from_numpy(shape),
                               torch.from_numpy(start))
    agg = CameraShardedAggregation.for_device_features(5, feats)
    t = lambda a: torch.from_numpy(a).to(cuda_dev)  # noqa: E731
    sl, sw = t(loc), t(wts)
    eager = agg(sl, sw, normalize=True, local_inputs=True)
    graph, out = agg.capture(sl, sw, normalize=True, local_inputs=True)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.allclose(out, eager, rtol=0, atol=1e-6 * float(eager.abs().max()))
    ref = mo.msda_dense_groups(table, tiles, shape, loc, wts, 4, normalize=True)
    assert float(np.abs(out.cpu().numpy() - ref).max()) <= 1e-4 * float(np.abs(ref).max())
    _, _, loc2, wts2 = helpers.make_dense(np.random.default_rng(22), bs=1, n_q=30, n_p=13, cams=5, n_levels=4,
                                          groups=8, channels=256, size_lo=8, size_hi=30)
    sl.copy_(t(loc2))
    sw.copy_(t(wts2))
    graph.replay()
    torch.cuda.synchronize()
    ref2 = mo.msda_dense_groups(table, tiles, shape, loc2, wts2, 4, normalize=True)
    assert float(np.abs(out.cpu().numpy() - ref2).max()) <= 1e-4 * float(np.abs(ref2).max())
    agg.close()
