"""Host/device time split of one net training step (dev tool).

    python tools/diag_step.py c3|c2
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2511_14852_b200 as ck  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda", 0)
dims = bench.layer_dims(wl)
layers = [ck.ChebyKANLayer(i, o, wl["degree"], lut_size=wl["lut_size"]) for i, o in dims]
model = torch.nn.Sequential(*layers).to(dev)
opt = ck.Adam(model.parameters(), lr=1e-4)
rows = wl["global_batch"]
x = torch.randn(rows, dims[0][0], device=dev)
tgt = torch.randn(rows, dims[-1][1], device=dev)


def step():
    y = model(x)
    loss = torch.nn.functional.mse_loss(y, tgt)
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
st0 = torch.cuda.memory_stats()
for phase in range(3):
    t0 = time.perf_counter()
    y = model(x)
    t1 = time.perf_counter()
    loss = torch.nn.functional.mse_loss(y, tgt)
    loss.backward()
    t2 = time.perf_counter()
    opt.step()
    opt.zero_grad(set_to_none=True)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"host fwd {1e3*(t1-t0):.2f} ms, bwd {1e3*(t2-t1):.2f}, opt {1e3*(t3-t2):.2f}, sync wait {1e3*(t4-t3):.2f}")
st1 = torch.cuda.memory_stats()
print("segment allocs during timed steps:", st1["segment.all.allocated"] - st0["segment.all.allocated"],
      "cudaMalloc retries:", st1["num_alloc_retries"] - st0["num_alloc_retries"])
from torch.profiler import profile, ProfilerActivity  # noqa: E402

with profile(activities=[ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=15))
