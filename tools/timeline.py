"""Device timeline of one decomposition (torch.profiler / CUPTI): kernel start, duration, stream.
Shows the critical path, the overlap of the two QR streams and host-launch gaps."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1810_07323_b200 as cg
from workloads import CONFIGS, make_device

name = sys.argv[1] if len(sys.argv) > 1 else "C2q1"
c = CONFIGS[name]
a = make_device(name)
ctx = cg.Context(0)
for i in range(3):
    cg.corutv(a, c.d, c.q, seed=cg.RngSeed(42, i), ctx=ctx)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    cg.corutv(a, c.d, c.q, seed=cg.RngSeed(42, 99), ctx=ctx)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
cpu = [e for e in prof.events() if e.name == "corutv" or "coru" in e.name]
print(f"{'start_us':>9} {'dur_us':>8}  stream  kernel")
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {getattr(e, 'device_resource_id', '?'):>6}  {e.name[:90]}")
print("device span us:", evs[-1].time_range.end - t0)
