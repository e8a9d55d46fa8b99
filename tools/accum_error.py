"""Accuracy vs reduction-chain length of the tcgen05 BF16x3 GEMMs (dev tool).

    python tools/accum_error.py            # driver: one subprocess per setting
    python tools/accum_error.py worker M   # one setting (env CK_GEMM_SPLITS)

The C4 layer (4096 -> 4096, d8, N = 32768): the forward reduces over
d * I = 32768 terms per output.  Rows 0..255 of an M-row batch (M = 256 or a
full 32768-row chunk) are compared with the float64 oracle; CK_GEMM_SPLITS
forces the number of reduction splits (fixed-order fp32 merge of partials).
Also the dC of a 32768-row chunk against a rank-1 dy (dC[k,o,i] = sum_b u_b
T_k(x_bi), the same for every o) computed in float64 -- the batch-long chain.
"""
import json
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(m):
    import torch

    import paper_2511_14852_b200 as ck
    from oracle import chebykan_oracle as orc

    dev = torch.device("cuda", 0)
    x0, c_jod, dy0 = orc.bench_inputs(256, 4096, 4096, 8, seed=3)
    vals, slopes, _ = orc.build_table(8, 32768)
    c_doj = orc.jod_to_doj(c_jod.astype(np.float64))
    cache_path = "/tmp/accum_oracle.npz"
    if os.path.exists(cache_path):
        wy = np.load(cache_path)["y"]
    else:
        wy = orc.layer_forward(x0, c_doj, vals, threads=orc.default_threads())
        np.savez(cache_path, y=wy)
    g = torch.Generator(device=dev).manual_seed(5)
    x = torch.rand(m, 4096, device=dev, generator=g) * 3 - 1.5
    x[:256] = torch.from_numpy(x0).to(dev)
    layer = ck.ChebyKANLayer(4096, 4096, 8, lut_size=32768).to(dev)
    with torch.no_grad():
        layer.coeff_doj.copy_(torch.from_numpy(c_doj.astype(np.float32)))
        y = layer(x)
    out = {"M": m, "splits": os.environ.get("CK_GEMM_SPLITS", "model"),
           "y_err": orc.normwise_err(y[:256].cpu().numpy(), wy)}
    if m >= 32768:
        # dC of the chunk for a rank-1 dy: u_b for every output column
        u = torch.randn(m, device=dev, generator=g)
        dy = u[:, None].expand(m, 4096).contiguous()
        layer.coeff_doj.grad = None
        xr = x.detach()
        with torch.enable_grad():
            layer(xr).backward(dy)
        dc = layer.coeff_doj.grad  # [9, 4096, 4096]
        # float64 reference: sum_b u_b T_k(x_bi) in row blocks
        t = torch.tanh(xr.double())
        phi = ck.expand(xr, ck.lut_build(ck.BasisKind.CHEBYSHEV, 8, 32768, device=dev))  # fp32 LUT values
        ref = torch.einsum("b,bik->ki", u.double(), phi.double())
        del t, phi
        err = ((dc.double() - ref[:, None, :]).abs().amax() / ref.abs().amax()).item()
        out["dC_rank1_err"] = err
    print(json.dumps(out), flush=True)


def main():
    rows = []
    for m in (256, 32768):
        for s in ("", "1", "2", "4", "8"):
            env = dict(os.environ)
            if s:
                env["CK_GEMM_SPLITS"] = s
            r = subprocess.run([sys.executable, __file__, "worker", str(m)], env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"M": m, "err": r.stderr[-500:]})
            print(line, flush=True)
            rows.append(json.loads(line))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/accum_error.json", "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "worker":
        worker(int(sys.argv[2]))
    else:
        main()
