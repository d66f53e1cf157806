"""Measurement tool: single-frame latency breakdown (C2): per-stage CUDA-event
times for F=1 and the host wall time of rg_range_frames."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_07980_b200 import ranger as rg, synth as S
from paper_2604_07980_b200.engine import FrameEngine, pack_detections
sc, cfg = S.scene_c2(seed=1, noise=2.0)
L, R = S.render_stereo_pair(sc)
dets = S.ground_truth_detections(sc)
ctx = rg.Context(0)
eng = FrameEngine(1920, 1080, cfg, len(dets), ctx=ctx)
dev = torch.device("cuda", 0)
dL = torch.from_numpy(L[None]).to(dev); dR = torch.from_numpy(R[None]).to(dev)
recs, offs = pack_detections([dets])
d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev); d_offs = torch.from_numpy(offs).to(dev)
out = torch.zeros(eng.out_stride * 32, dtype=torch.uint8, device=dev); cnt = torch.zeros(1, dtype=torch.int32, device=dev)
st = torch.cuda.Stream(dev)
for _ in range(20): eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
torch.cuda.synchronize()
ctx.reset_counters(); ctx.set_profiling(True)
N = 200
for _ in range(N): eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
torch.cuda.synchronize(); ctx.set_profiling(False)
ms, n, _ = ctx.counters()
print("per-frame stage ms:", {k: round(ms[i] / max(n[i], 1), 4) for i, k in enumerate(["census", "plan", "match", "agg"])})
wall = []
for _ in range(N):
    a = time.perf_counter(); eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream); st.synchronize()
    wall.append(time.perf_counter() - a)
print("wall p50 ms", round(1000 * statistics.median(wall), 4))
