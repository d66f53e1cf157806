"""SGM timing (measurement tool): rg_sgm_frames over device-resident C2 frames."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_07980_b200 import ranger as rg, synth as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nd = int(sys.argv[2]) if len(sys.argv) > 2 else 64
sc, _ = S.scene_c2(seed=1, noise=2.0)
L, R = S.render_stereo_pair(sc)
ctx = rg.Context(0)
dev = torch.device("cuda", 0)
dL = torch.from_numpy(np.stack([L] * n)).to(dev); dR = torch.from_numpy(np.stack([R] * n)).to(dev)
out = torch.zeros(n * L.size, dtype=torch.int16, device=dev)
p = rg.SgmParams(nd, 0, 8, 32).to_c()
st = torch.cuda.Stream(dev)
def run():
    ctx.check(rg.lib().rg_sgm_frames(ctx.handle, dL.data_ptr(), dR.data_ptr(), n, L.size, 1920, 1920, 1080,
                                     C.byref(p), out.data_ptr(), C.c_void_p(st.cuda_stream)))
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); run(); e1.record(st); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"SGM 1920x1080 nd={nd}: {ms:.3f} ms/frame, {1000/ms:.1f} frames/s, valid {(out.cpu().numpy() != -32768).mean():.3f}")
