"""Cost of the store GEMMs' accumulation segments (dev tool).

    python tools/seg_sweep.py [segs...]     # default: 0 16 32 64 128, twice, interleaved

For each CK_GEMM_SEG value (a subprocess each): one C4 training step
(4096 -> 4096, d8, N = 32768, one 32768-row chunk) repeated; the library's
per-class device timers give ms per GEMM launch, nvidia-smi the SM clock
during the run, so ms x MHz (= cycles) compares runs at different
power-capped clocks.  Accuracy: rows 0..255 of y against the float64 oracle.
"""
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker():
    import torch

    import paper_2511_14852_b200 as ck
    from oracle import chebykan_oracle as orc
    from paper_2511_14852_b200 import _lib

    dev = torch.device("cuda", 0)
    x0, c_jod, dy0 = orc.bench_inputs(256, 4096, 4096, 8, seed=3)
    c_doj = orc.jod_to_doj(c_jod.astype(np.float64))
    cache = "/tmp/seg_oracle.npz"
    if os.path.exists(cache):
        wy = np.load(cache)["y"]
    else:
        vals, _, _ = orc.build_table(8, 32768)
        wy = orc.layer_forward(x0, c_doj, vals, threads=orc.default_threads())
        np.savez(cache, y=wy)
    g = torch.Generator(device=dev).manual_seed(5)
    m = 32768
    x = torch.rand(m, 4096, device=dev, generator=g) * 3 - 1.5
    x[:256] = torch.from_numpy(x0).to(dev)
    dy = torch.randn(m, 4096, device=dev, generator=g)
    layer = ck.ChebyKANLayer(4096, 4096, 8, lut_size=32768).to(dev)
    with torch.no_grad():
        layer.coeff_doj.copy_(torch.from_numpy(c_doj.astype(np.float32)))
    xr = x.requires_grad_(True)

    def step():
        layer.coeff_doj.grad = None
        layer.bias.grad = None
        xr.grad = None
        y = layer(xr)
        y.backward(dy)
        return y

    for _ in range(2):
        y = step()
    torch.cuda.synchronize()
    err = orc.normwise_err(y[:256].detach().cpu().numpy(), wy)
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    _lib.timing_collect()
    _lib.timing_enable(True)
    reps = int(os.environ.get("SEG_REPS", "8"))
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_collect()
    smi.terminate()
    out = smi.communicate()[0]
    rows = [line.split(",") for line in out.strip().splitlines() if line.count(",") == 1]
    mhz = [float(a) for a, _ in rows if float(a) > 500]
    watts = [float(b) for a, b in rows if float(a) > 500]
    res = {"seg": os.environ.get("CK_GEMM_SEG", "default"), "y_err": err,
           "sm_mhz": statistics.median(mhz) if mhz else None, "watts": statistics.median(watts) if watts else None}
    for k in ("gemm_fwd", "gemm_dx", "gemm_dc"):
        ms, n = kt[k]
        res[k + "_ms"] = ms / max(1, n)
        if res["sm_mhz"]:
            res[k + "_mcyc"] = ms / max(1, n) * res["sm_mhz"] / 1e3
    print(json.dumps(res), flush=True)


def main():
    segs = sys.argv[1:] or ["0", "16", "32", "64", "128"]
    rows = []
    for rnd in range(2):
        for s in segs:
            env = dict(os.environ, CK_GEMM_SEG=s)
            r = subprocess.run([sys.executable, __file__, "worker"], env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"seg": s, "err": r.stderr[-400:]})
            print(line, flush=True)
            rows.append(json.loads(line))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "seg_sweep.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "worker":
        worker()
    else:
        main()
