"""rg_range_frames step time under different schedules (measurement tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_07980_b200 import ranger as rg, synth as S
from paper_2604_07980_b200.engine import FrameEngine, pack_detections
F = 256
sc, cfg = S.scene_c2(seed=1, noise=2.0)
L, R = S.render_stereo_pair(sc); dets = S.ground_truth_detections(sc)
ctx = rg.Context(0); eng = FrameEngine(1920, 1080, cfg, len(dets), ctx=ctx)
dev = torch.device("cuda", 0)
dL = torch.from_numpy(np.stack([L] * F)).to(dev); dR = torch.from_numpy(np.stack([R] * F)).to(dev)
recs, offs = pack_detections([dets] * F)
d_dets = torch.from_numpy(recs.view(np.uint8)).to(dev); d_offs = torch.from_numpy(offs).to(dev)
out = torch.zeros(F * eng.out_stride * 32, dtype=torch.uint8, device=dev); cnt = torch.zeros(F, dtype=torch.int32, device=dev)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
for ov in (False, True):
    ctx.set_overlap(ov)
    for _ in range(3): eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10): eng.range_device(dL, dR, d_dets, d_offs, out, cnt, stream=st.cuda_stream)
    e1.record(st); torch.cuda.synchronize()
    print(os.environ.get("RG_CHUNKS", "4"), os.environ.get("RG_CENSUS_PRIO", "lo"), "overlap" if ov else "serial", round(e0.elapsed_time(e1) / 10, 3), "ms/step")
