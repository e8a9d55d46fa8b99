"""Warm per-kernel device times of a CUDA-graph-replayed training step, from
CUPTI activity records (torch.profiler), in launch order (dev tool).  Unlike
an ncu launch list the kernels run back to back with warm caches and
programmatic dependent launch, as in bench.py's timed region.

    python tools/cupti_step.py c2|c3 [replays]
    python tools/cupti_step.py B I O degree [replays]   # one layer, x requires grad
"""
import collections
import os
import re
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2511_14852_b200 as ck  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)
argv = sys.argv[1:]
if argv[0] in bench.WORKLOADS:
    wl = bench.WORKLOADS[argv[0]]
    dims = bench.layer_dims(wl)
    d, rows = wl["degree"], wl["global_batch"]
    model = torch.nn.Sequential(*[ck.ChebyKANLayer(i, o, d, lut_size=wl["lut_size"]) for i, o in dims]).to(dev)
    x = torch.randn(rows, dims[0][0], device=dev)
    tgt = torch.randn(rows, dims[-1][1], device=dev)
    loss_fn = lambda y: ck.mse(y, tgt)  # noqa: E731 (as bench.py)
    reps = int(argv[1]) if len(argv) > 1 else 10
else:
    b, i, o, d = (int(a) for a in argv[:4])
    model = ck.ChebyKANLayer(i, o, d, lut_size=32768).to(dev)
    x = (torch.rand(b, i, device=dev) * 3 - 1.5).requires_grad_(True)
    dy = torch.randn(b, o, device=dev)
    loss_fn = lambda y: (y * dy).sum()  # noqa: E731
    reps = int(argv[4]) if len(argv) > 4 else 10
opt = ck.Adam(model.parameters(), lr=1e-4, capturable=True)


def step():
    if x.requires_grad:
        x.grad = None
    loss_fn(model(x)).backward()
    opt.step()
    opt.zero_grad(set_to_none=True)


side = torch.cuda.Stream(device=dev)
side.wait_stream(torch.cuda.current_stream(dev))
with torch.cuda.stream(side):
    for _ in range(3):
        step()
torch.cuda.current_stream(dev).wait_stream(side)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(reps):
    g.replay()
ev[1].record()
torch.cuda.synchronize()
step_ms = ev[0].elapsed_time(ev[1]) / reps
if os.environ.get("NO_CUPTI"):  # under ncu (CUPTI has one subscriber)
    print(f"step {step_ms * 1000:.1f} us (graph replay, CUDA events)")
    sys.exit(0)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        g.replay()
    torch.cuda.synchronize()
kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern.sort(key=lambda e: e.time_range.start)
per = len(kern) // reps
print(f"step {step_ms * 1000:.1f} us (graph replay, CUDA events); {per} kernels per step")
# With programmatic dependent launch a kernel's recorded start is its early
# launch (it then waits for its predecessor), so durations overlap; the
# critical-path cost of kernel j is end_j - end_{j-1}.
acc = collections.OrderedDict()
for j, e in enumerate(kern[: per * reps]):
    name = re.sub(r"\(anonymous namespace\)::", "", e.name)
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*", "", name)[:70]
    prev_end = kern[j - 1].time_range.end if j > 0 and j % per else e.time_range.start
    key = (j % per, name)
    a = acc.setdefault(key, [0.0, 0.0])
    a[0] += (e.time_range.end - prev_end) / reps
    a[1] += e.time_range.elapsed_us() / reps
span = (kern[per * reps - 1].time_range.end - kern[0].time_range.start) / reps
for (j, name), (inc, dur) in acc.items():
    print(f"{j:3d} {inc:8.2f} us (recorded {dur:7.2f})  {name}")
print(f"profiled span {span:.1f} us per step (critical-path increments sum to it, less the gaps between replays)")
