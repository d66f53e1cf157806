"""Device frame source timing (measurement tool): rg_render_frames_device over
F distinct C2 scenes (noise 2.0), CUDA events, vs the host renderer."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_07980_b200 import ranger as rg, synth as S

F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = rg.Context(0)
scenes = [S.scene_c2(seed=1 + i, noise=2.0)[0] for i in range(F)]
dev = torch.device("cuda", 0)
L = torch.empty((F, 1080, 1920), dtype=torch.uint8, device=dev)
R = torch.empty_like(L)
S.render_frames_device(ctx, scenes[:8], L, R)
torch.cuda.synchronize()
for noise in (2.0, 0.0):
    for sc in scenes:
        sc.noise_sigma = noise
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    S.render_frames_device(ctx, scenes, L, R, stream=torch.cuda.current_stream().cuda_stream)
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = a.elapsed_time(b)
    print(f"noise {noise}: {F} C2 frames {ms:.2f} ms device ({F / ms * 1e3:.0f} frames/s), wall {wall * 1e3:.1f} ms")
t0 = time.perf_counter()
S.render_stereo_pair(S.scene_c2(seed=1, noise=2.0)[0])
print(f"host renderer: one C2 frame {1e3 * (time.perf_counter() - t0):.1f} ms ({os.cpu_count()} cpus)")
