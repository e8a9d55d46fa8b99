"""Sustained throughput of cuBLASLt int8 (torch._int_mm) vs bf16 GEMM under the
power cap -- decides whether an int8-slice (Ozaki-style) contraction would
beat BF16x3 on this part.  Prints TOPS/TFLOPS and median SM clock per mode."""
import subprocess
import time

import torch


def run(fn, flops, secs=6.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    # time one call to size the batch of launches
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    n = max(10, int(secs * 1e3 / a.elapsed_time(b)))
    log = open("/tmp/clk.csv", "w")
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=log)
    time.sleep(0.3)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    smi.terminate()
    smi.wait()
    ms = a.elapsed_time(b)
    rows = [l.split(",") for l in open("/tmp/clk.csv").read().splitlines() if "," in l]
    rows = [(float(r[0]), float(r[1])) for r in rows][len(rows) // 3:]
    mhz = sorted(r[0] for r in rows)[len(rows) // 2]
    w = sorted(r[1] for r in rows)[len(rows) // 2]
    return flops * n / (ms / 1e3) / 1e12, mhz, w


N = 8192
dev = torch.device("cuda")
A16 = torch.randn(N, N, device=dev, dtype=torch.bfloat16)
B16 = torch.randn(N, N, device=dev, dtype=torch.bfloat16)
A8 = torch.randint(-127, 127, (N, N), device=dev, dtype=torch.int8)
B8 = torch.randint(-127, 127, (N, N), device=dev, dtype=torch.int8).t().contiguous().t()
f = 2 * N ** 3
for name, fn in (("bf16", lambda: torch.matmul(A16, B16)), ("int8", lambda: torch._int_mm(A8, B8)),
                 ("bf16", lambda: torch.matmul(A16, B16)), ("int8", lambda: torch._int_mm(A8, B8))):
    t, mhz, w = run(fn, f)
    print(f"{name}: {t:8.1f} T(FL)OPS sustained, SM {mhz:.0f} MHz, {w:.0f} W", flush=True)
