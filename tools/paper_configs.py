"""B200 timings at the reference's three paper configurations (dev tool).

    python tools/paper_configs.py     # -> gpurun_out/paper_configs.json (+ markdown table on stdout)

perf.run_bench (the reference's perf.py:225-275 protocol: median of reps
after warm-ups) on perf.paper_configs() (perf.py:137-143) for the five
kernel versions, plus the prepared-coefficient LUT path replayed from a
captured CUDA graph (these layers are launch-bound).  The A100 V5 numbers
are PAPER.md:873-881 as quoted in SURVEY.md section 6.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

A100_V5 = {(128, 40, 256, 8): (0.046, 0.123), (64, 256, 512, 15): (0.376, 1.006), (32, 512, 1024, 24): (1.580, 4.500)}


def graph_time(cfg, reps=200):
    import torch

    import paper_2511_14852_b200 as ck
    from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw, forward_raw
    from paper_2511_14852_b200.perf import _bench_inputs

    dev = torch.device("cuda", 0)
    x, c_jod, dy = _bench_inputs(cfg, 0, dev)
    lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, cfg.degree, 32768, device=dev)
    prep = PreparedCoeff(ck.reorder_to_doj(c_jod).data)
    nbytes = ck.kernels.basis_cache_bytes(cfg.batch, cfg.d_in, cfg.d_out, cfg.degree + 1)
    cache = torch.empty(max(1, nbytes), dtype=torch.uint8, device=dev) if nbytes else None

    def fwd():
        forward_raw(x, prep, lut, None, cache)

    def bwd():
        backward_raw(x, dy, prep, lut, True, want_db=False, cache=cache)

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fwd()
            bwd()
    torch.cuda.current_stream().wait_stream(side)
    gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf):
        fwd()
    with torch.cuda.graph(gb):
        bwd()
    for _ in range(10):
        gf.replay()
        gb.replay()
    torch.cuda.synchronize()
    out = []
    for g in (gf, gb):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            g.replay()
        ev[1].record()
        torch.cuda.synchronize()
        out.append(ev[0].elapsed_time(ev[1]) / reps)
    return out


def main():
    import paper_2511_14852_b200 as ck

    res = ck.run_bench(ck.paper_configs(), list(ck.perf.KERNEL_VERSIONS), reps=50, warmups=10)
    rows = []
    for r in res:
        c = r.config
        rows.append({"config": [c.batch, c.d_in, c.d_out, c.degree], "version": r.version, "fwd_ms": r.fwd_ms,
                     "bwd_ms": r.bwd_ms, "samples_per_s": r.samples_per_s, "mode": "eager (run_bench)"})
    for c in ck.paper_configs():
        f, b = graph_time(c)
        rows.append({"config": [c.batch, c.d_in, c.d_out, c.degree], "version": "fused-lut+reorder", "fwd_ms": f,
                     "bwd_ms": b, "samples_per_s": c.batch / ((f + b) / 1e3), "mode": "CUDA graph replay"})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "paper_configs.json"), "w") as fh:
        json.dump(rows, fh, indent=1)
    print("| (B, I, O, d) | version | mode | fwd ms | bwd ms | A100 V5 fwd / bwd ms (PAPER.md:873-881) |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        a = A100_V5.get(tuple(r["config"]))
        print(f"| {tuple(r['config'])} | {r['version']} | {r['mode']} | {r['fwd_ms']:.4f} | {r['bwd_ms']:.4f} | "
              f"{a[0]} / {a[1]} |")


if __name__ == "__main__":
    main()
