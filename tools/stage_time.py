"""Stage timing (measurement tool): rg_range_frames over F device-resident
C2 frames (device-rendered, distinct seeds), per-stage CUDA events, mean of
N launches.  RG_LIB_PATH selects a library variant.
  python tools/stage_time.py [F] [N] [scene: c2 (default) | c3 | c1]"""
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
SC = {"c2": S.scene_c2, "c3": S.scene_c3, "c1": S.scene_c1}[sys.argv[3] if len(sys.argv) > 3 else "c2"]
scenes = [SC(seed=1 + i, noise=2.0)[0] for i in range(F)]
dets, cfg = S.ground_truth_detections(scenes[0]), SC(seed=1)[1]
W, H = scenes[0].width, scenes[0].height
dL = torch.empty((F, H, W), dtype=torch.uint8, device=dev)
dR = torch.empty_like(dL)
S.render_frames_device(ctx, scenes, dL, dR)
eng = FrameEngine(W, H, cfg, len(dets), S.F_PX, S.BASELINE_M, ctx=ctx)
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
print(f"{tag} F={F} census {ms[0] / N:.4f} plan {ms[1] / N:.4f} match {ms[2] / N:.4f} "
      f"agg {ms[3] / N:.4f} ms/step; evals/frame {ev / (N * F):.0f}; "
      f"match {ev / N / (ms[2] / N * 1e-3) / 1e12:.3f} Tevals/s; stable={bool(torch.equal(ref, out))}")
