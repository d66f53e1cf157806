"""Measurement tool: 256 device-resident C2 frames ranged as one batch vs as
consecutive chunks of C frames (asynchronous batches on one stream): does a
census -> matcher sequence per chunk whose rasters fit in L2 pay?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_07980_b200 import ranger as rg, synth as S
from paper_2604_07980_b200.engine import FrameEngine, pack_detections

F = 256
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
out = torch.zeros(F * eng.out_stride * 32, dtype=torch.uint8, device=dev)
cnt = torch.zeros(F, dtype=torch.int32, device=dev)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
for C in (256, 128, 64, 32, 16, 8):
    d_offs = torch.from_numpy(pack_detections([dets] * C)[1]).to(dev)

    def run():
        for c0 in range(0, F, C):
            eng.range_device(dL[c0:c0 + C], dR[c0:c0 + C], d_dets, d_offs, out[c0 * eng.out_stride * 32:],
                             cnt[c0:], stream=st.cuda_stream, sync=False)
    for _ in range(3):
        run()
    ctx.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        run()
    e1.record(st)
    assert ctx.sync() == 0
    torch.cuda.synchronize()
    print(f"chunk {C:4d}: {e0.elapsed_time(e1) / 10:.3f} ms per 256 frames")
