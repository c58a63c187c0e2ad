# compute-sanitizer workload: one small call of every production kernel (exact / fast / exact_half CSR,
# dense fast / fast_h2 / exact incl. the camera-group split, fused projection, OAE (one CTA per query and per camera
# group), visibility, painting, association, the peer-memory exchange) in f32 / f16 / bf16.
# Run: compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_workload.py
# Small invocations of every production kernel, for compute-sanitizer runs.
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import __graft_entry__ as g
g.smoke()  # exact CSR (plan + gather) + dense FAST
from paper_2601_10819_b200 import ops
from paper_2601_10819_b200.workload import BenchWorkload, generate_workload
dev = torch.device("cuda", 0)
wl = BenchWorkload(cameras=2, levels=4, channels=256, queries=16, points_per_query=13, level0_size=(32, 88))
gw = generate_workload(wl)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
for dt in (torch.float32, torch.float16, torch.bfloat16):
    feats = ops.DeviceFeatures(t(gw.table).to(dt), t(gw.spatial_shape), t(gw.tile_start.reshape(2, 4)))
    for prec in ("exact", "fast"):
        ops.msda_csr(feats, t(gw.offsets), t(gw.camera_ids), t(gw.levels), t(gw.us), t(gw.vs), t(gw.weights), precision=prec)
    if dt is torch.float16:
        ops.msda_csr(feats, t(gw.offsets), t(gw.camera_ids), t(gw.levels), t(gw.us), t(gw.vs), t(gw.weights), precision="exact_half")
    rng = np.random.default_rng(1)
    loc = t(rng.uniform(0, 1, (1, 16, 13, 2, 2)).astype(np.float32))
    w = t(rng.uniform(0.01, 1, (1, 16, 13, 2, 4, 8)).astype(np.float32))
    for prec in ("fast", "fast_h2", "exact"):
        if prec == "fast_h2" and dt is not torch.float16:
            continue
        # normalize=False: the fused one-pass EXACT kernel; f16/bf16 FAST: staged coarse levels (TMA) + fine gather
        for norm in (True, False):
            ops.deformable_aggregation(feats, None, None, loc, w, precision=prec, normalize=norm, check=True)
    K = np.array([[300.0, 300.0, 352.0, 128.0]] * 2)
    R = np.stack([np.eye(3), np.eye(3)]).reshape(2, 9)
    T = np.array([[0.0, 0.0, 10.0], [0.0, 0.0, 12.0]])
    cams = ops.Cameras(K, R, T, device=dev)
    anchors = torch.zeros((1, 16, 10), device=dev)
    anchors[..., 3:6] = torch.tensor([0.6, 0.6, 1.8])
    offs = np.zeros((6, 3), np.float32)
    wp = t(rng.uniform(0.01, 1, (1, 16, 13, 2, 4, 8)).astype(np.float32))
    ops.msda_dense_project(feats, anchors, offs, cams, [4.0, 8.0, 16.0, 32.0], wp, check=True)
    desc = torch.randn((16, 256), device=dev)
    vis = torch.rand((16, 2), device=dev)
    mem = torch.nn.functional.normalize(torch.randn((16, 256), device=dev), dim=1)
    ops.oae_pool(feats, anchors[0], offs, cams, [4.0, 8.0, 16.0, 32.0], desc, vis, mem)
# more than one camera group: the dense pipelined gather's split path (red.add partials + group normalise,
# also with the caller's weight sums) and the OAE (query, camera group) CTAs + finishing kernel
wl9 = BenchWorkload(cameras=9, levels=4, channels=256, queries=8, points_per_query=13, level0_size=(32, 88))
gw9 = generate_workload(wl9)
rng = np.random.default_rng(2)
K9 = np.array([[300.0, 300.0, 352.0, 128.0]] * 9)
R9 = np.stack([np.eye(3)] * 9).reshape(9, 9)
T9 = np.array([[0.0, 0.0, 10.0 + c] for c in range(9)])
cams9 = ops.Cameras(K9, R9, T9, device=dev)
for dt in (torch.float32, torch.float16, torch.bfloat16):
    f9 = ops.DeviceFeatures(t(gw9.table).to(dt), t(gw9.spatial_shape), t(gw9.tile_start.reshape(9, 4)))
    loc9 = t(rng.uniform(0, 1, (1, 8, 13, 9, 2)).astype(np.float32))
    w9 = t(rng.uniform(0.01, 1, (1, 8, 13, 9, 4, 8)).astype(np.float32))
    for prec in ("fast", "fast_h2"):
        if prec == "fast_h2" and dt is not torch.float16:
            continue
        ops.deformable_aggregation(f9, None, None, loc9, w9, precision=prec, normalize=True, check=True)
    ops.deformable_aggregation_partial(f9, loc9, w9, precision="fast")
    a9 = torch.zeros((8, 10), device=dev)
    a9[:, 3:6] = torch.tensor([0.6, 0.6, 1.8])
    ops.oae_pool(f9, a9, np.zeros((6, 3), np.float32), cams9, [4.0, 8.0, 16.0, 32.0], torch.randn((8, 256), device=dev),
                 torch.rand((8, 9), device=dev),
                 torch.nn.functional.normalize(torch.randn((8, 256), device=dev), dim=1))
# peer-memory exchange (world 1: own buffer only), two epochs so both halves are used
from paper_2601_10819_b200.dist import PeerExchange
px = PeerExchange(16, 256, 8, dev)
for _ in range(2):
    px.allreduce_normalize(torch.rand((16, 256), device=dev), torch.rand((16, 8), device=dev) + 0.5, True)
px.allreduce_normalize(torch.rand((16, 256), device=dev), torch.rand((16, 8), device=dev) + 0.5, False)
px.close()
ops.visibility(cams, [[704, 256]] * 2, [[0, 0, 0, 1, 1, 1, 0], [0.5, 0, 1, 1, 1, 1, 0.3]], grid=16)
sc = ops.PaintScene(cams, [[704, 256]] * 2, [8.0, 16.0], 32, [[0, 0, 0, 1, 1, 1, 0], [0.5, 0, 1, 1, 1, 1, 0.3]], 1,
                    np.ones((1, 32)) / np.sqrt(32))
sc.run(seed=3)
sc.run(background=np.zeros((sc.rows, 32)))
ops.association_cost(np.zeros((20, 3)), np.ones((17, 3)), np.random.rand(20, 130), np.random.rand(17, 130), device=dev)
# bilinear_sample through the host entry point (pageable grid: copied; a reused large grid: page-locked, read in place)
from paper_2601_10819_b200 import features as F
pyr = F.FeaturePyramid(0, [F.FeatureGrid(stride=4.0, values=np.random.rand(9, 7, 6).astype(np.float32))])
for u, v in [(0.3, 0.2), (-1.5, 3.0), (6.0, 8.0)]:
    F.bilinear_sample(pyr, 0, u, v)
big = F.FeaturePyramid(0, [F.FeatureGrid(stride=4.0, values=np.random.rand(512, 1024, 4).astype(np.float32))])
for _ in range(3):
    F.bilinear_sample(big, 0, 100.5, 200.25)
torch.cuda.synchronize()
print("sanitizer workload done")
