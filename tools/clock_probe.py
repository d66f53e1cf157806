"""Measurement tool: exercise bench.ClockSampler on the GPU box."""
import faulthandler, sys, os, time
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print("props", torch.cuda.get_device_properties(0))
c = bench.ClockSampler(0)
c.start()
print("nvml", c.nvml is not None, "rows", len(c.rows), flush=True)
x = torch.randn(8192, 8192, device="cuda")
for _ in range(50):
    x = x @ x
    x = x / x.norm()
torch.cuda.synchronize()
print(c.stop(), flush=True)
