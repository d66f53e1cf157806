"""Stage timing (measurement tool): rg_range_frames over F device-resident
C2 frames (device-rendered, distinct seeds), per-stage CUDA events, mean of
N launches.  RG_LIB_PATH selects a library variant.
  python tools/stage_time.py [F] [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_07980_b200 import ranger as rg, synth as S
from paper_2604_07980_b200.engine import FrameEngine, pack_detections

F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = rg.Context(0)
dev = torch.device("cuda", 0)
scenes = [S.scene_c2(seed=1 + i, noise=2.0)[0] for i in range(F)]
dets, cfg = S.ground_truth_detections(scenes[0]), S.scene_c2(seed=1)[1]
dL = torch.empty((F, 1080, 1920), dtype=torch.uint8, device=dev)
dR = torch.empty_like(dL)
S.render_frames_device(ctx, scenes, dL, dR)
eng = FrameEngine(1920, 1080, cfg, len(dets), S.F_PX, S.BASELINE_M, ctx=ctx)
recs, offs = pack_detections([dets] * F)
d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev)
d_offs = torch.from_numpy(offs).to(dev)
out = torch.zeros(F * eng.out_stride * 32, dtype=torch.uint8, device=dev)
cnt = torch.zeros(F, dtype=torch.int32, device=dev)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
for _ in range(3):
    eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
torch.cuda.synchronize()
ref = out.clone()
ctx.reset_counters()
ctx.set_profiling(True)
for _ in range(N):
    eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
torch.cuda.synchronize()
ctx.set_profiling(False)
ms, n, _ = ctx.counters()
ev, _ = ctx.work()
tag = (os.environ.get("RG_LIB_PATH") or "x/base/x").split("/")[-2]
print(f"{tag} F={F} census {ms[0] / n[0]:.4f} plan {ms[1] / n[1]:.4f} match {ms[2] / n[2]:.4f} "
      f"agg {ms[3] / n[3]:.4f} ms/launch; evals/frame {ev / (N * F):.0f}; "
      f"match {ev / N / (ms[2] / n[2] * 1e-3) / 1e12:.3f} Tevals/s; stable={bool(torch.equal(ref, out))}")
