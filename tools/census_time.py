"""Census-only timing (measurement tool): K1 over 256 device-resident C2 frames,
CUDA events, best of N; run with RG_LIB_PATH to compare library variants."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_07980_b200 import ranger as rg
from paper_2604_07980_b200.engine import FrameEngine, pack_detections, OUT_DTYPE
from paper_2604_07980_b200 import synth as S
F = 256
sc, cfg = S.scene_c2(seed=1, noise=2.0)
L, R = S.render_stereo_pair(sc)
dets = S.ground_truth_detections(sc)
ctx = rg.Context(0)
eng = FrameEngine(1920, 1080, cfg, len(dets), ctx=ctx)
dev = torch.device("cuda", 0)
dL = torch.from_numpy(np.stack([L] * F)).to(dev); dR = torch.from_numpy(np.stack([R] * F)).to(dev)
recs, offs = pack_detections([dets] * F)
d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev); d_offs = torch.from_numpy(offs).to(dev)
out = torch.zeros(F * eng.out_stride * 32, dtype=torch.uint8, device=dev); cnt = torch.zeros(F, dtype=torch.int32, device=dev)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
for _ in range(3): eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
torch.cuda.synchronize()
ctx.reset_counters(); ctx.set_profiling(True)
for _ in range(20): eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
torch.cuda.synchronize(); ctx.set_profiling(False)
ms, n, _ = ctx.counters()
print((os.environ.get("RG_LIB_PATH") or "x/base/x").split("/")[-2], "census ms/launch", round(ms[0] / n[0], 4), "match", round(ms[2] / n[2], 4))
