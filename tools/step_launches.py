"""One eager training step inside a cudaProfilerStart/Stop range, for
`ncu --profile-from-start off` launch lists (dev tool).

    python tools/step_launches.py c2|c3          # bench.py's net workloads
    python tools/step_launches.py B I O degree   # one layer (x requires grad)
"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2511_14852_b200 as ck  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)
if sys.argv[1] in bench.WORKLOADS:
    wl = bench.WORKLOADS[sys.argv[1]]
    dims = bench.layer_dims(wl)
    d, rows = wl["degree"], wl["global_batch"]
    model = torch.nn.Sequential(*[ck.ChebyKANLayer(i, o, d, lut_size=wl["lut_size"]) for i, o in dims]).to(dev)
    x = torch.randn(rows, dims[0][0], device=dev)
    tgt = torch.randn(rows, dims[-1][1], device=dev)
    loss_fn = lambda y: torch.nn.functional.mse_loss(y, tgt)  # noqa: E731
else:
    b, i, o, d = (int(a) for a in sys.argv[1:5])
    model = ck.ChebyKANLayer(i, o, d, lut_size=32768).to(dev)
    x = (torch.rand(b, i, device=dev) * 3 - 1.5).requires_grad_(True)
    dy = torch.randn(b, o, device=dev)
    loss_fn = lambda y: (y * dy).sum()  # noqa: E731
opt = ck.Adam(model.parameters(), lr=1e-4)


def step():
    if x.requires_grad:
        x.grad = None
    loss_fn(model(x)).backward()
    opt.step()
    opt.zero_grad(set_to_none=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
