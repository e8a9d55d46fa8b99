#!/usr/bin/env python
"""Benchmark of the fused ChebyKAN layer on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c1] [--sweep]

Default workload (BASELINE.json configs[4], "C4"): data-parallel ChebyKAN
training 4096->4096, degree 8, LUT N=32768, global batch 262144 rows sharded
contiguously over the ranks (strong scaling; at N=1 one GPU runs all rows).
One step = forward + backward (dC, db, dX) + allreduce of dC/db (N>1) +
Adam update (+ the coefficient re-split the next forward needs), all on
synthetic data of the named shapes with random-init weights.

One JSON line on rank 0: ``value`` = training samples/s of the whole job,
device-timed (CUDA events, barrier + synchronize on both sides, max over
ranks), inputs resident in HBM (each rank's x shard is 4.3 GB at N=1, far
larger than the 126 MB L2, so no flush is needed).  ``e2e`` repeats the step
through the public module API with the step's x/dy copied from pinned host
memory and the loss read back every step.  ``roofline`` is the dominant
kernel (the tcgen05 BF16x3 GEMM family) timed live by the library's CUDA
event timers inside the timed region.  ``cpu_baseline`` is the oracle port
of the reference's CPU path on a bounded row sample (rank 0, N=1 only).

``--impl reference`` times the reference's CPU algorithm (oracle port; the
Python reference itself cannot travel to the GPU box) on the host cores.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "c4": dict(name="C4 DP ChebyKAN training 4096->4096 d8, global batch 262144", d_in=4096, d_out=4096,
               degree=8, global_batch=262144, lut_size=32768),
    "c1": dict(name="C1 ChebyKAN layer 4096->4096 d8, batch 16384 per GPU", d_in=4096, d_out=4096, degree=8,
               global_batch=16384, lut_size=32768, weak=True),
    "c2": dict(name="C2 tabular ChebyKAN net [64->512->512->1] d5, MSE, batch 16384", layers=[64, 512, 512, 1],
               degree=5, global_batch=16384, lut_size=32768),
    "c3": dict(name="C3 speech ChebyKAN FFN [257->512->512->257] d15, MSE, 64x500 frames", layers=[257, 512, 512, 257],
               degree=15, global_batch=32000, lut_size=32768),
}
METRIC = "ChebyKAN training (fwd+bwd+dC allreduce+Adam) samples/s"
METRIC_NET = "ChebyKAN net training (fwd+bwd+allreduce+Adam) samples/s"
CPU_SAMPLE_ROWS = 128      # oracle rows timed for cpu_baseline (~10-20 s of CPU work)
REF_STEP_ROWS = 64         # oracle rows per --impl reference step


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]),
                    bf16_sus=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, source="fallback (B200_PROFILING.md)")


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md recipe)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = pathlib.Path(f"/tmp/ck_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags) if f.lower() == "active"})
        loaded = [r[0] for r in rows if r[0] > 500] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU legs (oracle = test infrastructure, used here only as the baseline)

def layer_dims(wl):
    if "layers" in wl:
        return list(zip(wl["layers"][:-1], wl["layers"][1:]))
    return [(wl["d_in"], wl["d_out"])]


def cpu_info():
    """CPU model, numpy version and BLAS library of this host."""
    import platform

    import numpy as np

    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info

        libs = [f"{i.get('internal_api')} {i.get('version')}" for i in threadpool_info() if i.get("user_api") == "blas"]
        blas = ", ".join(libs) or None
    except Exception:  # noqa: BLE001 (informational only)
        blas = None
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def cpu_reference_time(rows: int, wl: dict, reps: int = 1, warmup: int = 0, mode: str = "tiles",
                       keep_outputs: bool = False):
    """Oracle port of the reference's fused_forward/backward_fused over the
    workload's layers (a net's layers run back to back, forward then backward).

    ``mode`` is one of the reference's two threading modes (BASELINE.md 4,
    perf.py:225-275): "tiles" = BLAS single-threaded, tile tasks on every
    core (POLYKAN_WORKERS = nproc); "blas" = one tile-task worker, BLAS on
    every core.  Returns (per-rep seconds, threads, layer inputs and the last
    rep's outputs if keep_outputs)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import chebykan_oracle as orc

    threads = os.cpu_count() or 1
    vals, slopes, _ = orc.build_table(wl["degree"], wl["lut_size"])
    layers = []
    for li, (i, o) in enumerate(layer_dims(wl)):
        x, c_jod, dy = orc.bench_inputs(rows, i, o, wl["degree"], seed=3 + li)
        layers.append((x, orc.jod_to_doj(c_jod.astype(np.float64)), dy))
    workers = threads if mode == "tiles" else 1
    times, outs = [], None
    with threadpool_limits(1 if mode == "tiles" else threads):
        for it in range(warmup + reps):
            t0 = time.perf_counter()
            ys = [orc.layer_forward(x, c_doj, vals, threads=workers) for x, c_doj, _ in layers]
            grads = [orc.layer_backward(x, c_doj, dy, vals, slopes, threads=workers)
                     for x, c_doj, dy in reversed(layers)][::-1]
            if it >= warmup:
                times.append(time.perf_counter() - t0)
            outs = (ys, grads)
    return times, threads, (layers if keep_outputs else None), (outs if keep_outputs else None)


def cpu_baseline(wl, rows):
    """BASELINE.md section 4 protocol on this host: both threading modes,
    median of reps after a warm-up, the better mode reported.  The tile-task
    mode (the faster one at these shapes) runs 3 reps on `rows` rows; the
    BLAS-threaded mode, several times slower here, 1 rep on rows/4 rows so
    the leg stays within ~30 s of CPU work."""
    rate = {}
    layers = outs = None
    for mode, n, reps in (("tiles", rows, 3), ("blas", max(1, rows // 4), 1)):
        times, threads, lay, out = cpu_reference_time(n, wl, reps=reps, warmup=1, mode=mode,
                                                      keep_outputs=mode == "tiles")
        rate[mode] = n / statistics.median(times)
        if lay is not None:
            layers, outs = lay, out
    best = max(rate, key=rate.get)
    return {
        "value": rate[best], "unit": "samples/s", "cores": threads, "kind": "port",
        "sample": (f"{rows} rows of {layer_dims(wl)} d{wl['degree']} N={wl['lut_size']}, fwd+bwd (no optimizer); "
                   f"oracle port of polykan LUT-mode fused_forward/backward_fused, f64 NumPy; median of 3 reps "
                   f"after 1 warm-up; the better of the two threading modes"),
        "threading_modes_samples_per_s": {
            "tiles (BLAS 1 thread, tile tasks on all cores)": rate["tiles"],
            "blas (1 tile worker, BLAS on all cores; rows/4, 1 rep)": rate["blas"]},
        "best_mode": best, **cpu_info(),
    }, layers, outs


def gpu_parity(wl, layers, outs):
    """Feed the cpu_baseline rows' exact inputs through the GPU module path
    (one chunk, and 8 chunks so dC accumulates like the full batch does) and
    compare with the oracle's outputs: normwise max|got-want|/max|want|."""
    import numpy as np
    import torch

    import paper_2511_14852_b200 as ck
    from oracle import chebykan_oracle as orc

    dev = torch.device("cuda", torch.cuda.current_device())
    ys, grads = outs
    worst = {"y": 0.0, "dX": 0.0, "dC": 0.0, "db": 0.0}
    rows = layers[0][0].shape[0]
    for (x, c_doj, dy), wy, (wdc, wdx, wdb) in zip(layers, ys, grads):
        i, o = x.shape[1], dy.shape[1]
        layer = ck.ChebyKANLayer(i, o, wl["degree"], lut_size=wl["lut_size"]).to(dev)
        with torch.no_grad():
            layer.coeff_doj.copy_(torch.from_numpy(c_doj.astype(np.float32)))
        for chunk in (0, max(1, rows // 8)):
            layer.zero_grad(set_to_none=True)
            xt = torch.from_numpy(x).to(dev).requires_grad_(True)
            with ck.chunk_rows(chunk):
                y = layer(xt)
                y.backward(torch.from_numpy(dy).to(dev))
            torch.cuda.synchronize(dev)
            got = {"y": (y.detach(), wy), "dX": (xt.grad, wdx), "dC": (layer.coeff_doj.grad, wdc),
                   "db": (layer.bias.grad, wdb)}
            for k, (g, w) in got.items():
                worst[k] = max(worst[k], orc.normwise_err(g.cpu().numpy(), w))
        del layer
    return {"rows": rows, "chunk_rows": [min(rows, 32768), max(1, rows // 8)], "normwise_max": worst,
            "tol": 1e-4, "pass": all(v <= 1e-4 for v in worst.values()),
            "against": "oracle (float64 restatement of kernels.py:351-447) on the cpu_baseline sample's inputs"}


def run_reference_arm(args, wl):
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    times, threads, _, _ = cpu_reference_time(REF_STEP_ROWS, wl, reps=args.steps, warmup=args.warmup)
    t = statistics.median(times)
    value = REF_STEP_ROWS / t
    sample = (f"{REF_STEP_ROWS} rows of {layer_dims(wl)} d{wl['degree']} N={wl['lut_size']} fwd+bwd per "
              f"step; oracle port of polykan fused_forward/backward_fused (LUT mode, f64 NumPy), "
              f"{threads} tile-task threads, BLAS 1 thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "global_batch": wl["global_batch"], "layers": layer_dims(wl),
                   "degree": wl["degree"], "lut_size": wl["lut_size"],
                   "parallelism": "host threads", "sample_rows_per_step": REF_STEP_ROWS},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm

def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2511_14852_b200 as ck
    from paper_2511_14852_b200 import _lib

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # CK_BENCH_BACKEND=gloo lets N ranks share fewer GPUs (plumbing checks on a
    # 1-GPU box; NCCL refuses two ranks per device); the default is NCCL
    backend = os.environ.get("CK_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_ALGO", "Ring")  # fixed reduction order -> reproducible dC
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    if _lib.lib().ck_device_supported(local) != 1:
        raise SystemExit(f"device {torch.cuda.get_device_name(local)} is not sm_100 (B200)")

    d = wl["degree"]
    dims = layer_dims(wl)
    is_net = "layers" in wl
    I, O = dims[0][0], dims[-1][1]
    if wl.get("weak"):
        gb = wl["global_batch"] * world
        a, b = rank * wl["global_batch"], (rank + 1) * wl["global_batch"]
    else:
        gb = wl["global_batch"]
        a, b = ck.shard_bounds(gb, rank, world)
    rows = b - a

    torch.manual_seed(1234)  # identical synthetic weights on every rank
    layers = [ck.ChebyKANLayer(i, o, d, lut_size=wl["lut_size"]) for i, o in dims]
    model = (torch.nn.Sequential(*layers) if is_net else layers[0]).to(dev)
    # graphs on one GPU only (the N>1 exchange brackets its kernel with host barriers)
    use_graph = (args.graph if args.graph is not None else is_net) and world == 1
    # ck_adam_step (reference adam_step rule); device-side step counter when captured
    opt = ck.Adam(model.parameters(), lr=1e-4, capturable=use_graph)
    reducer, reducer_kind = None, None
    if world > 1:
        params = ck.chebykan_parameters(model)
        if args.reducer == "peer":
            try:
                # the library's fixed-order peer-memory allreduce (CUDA IPC over NVLink)
                reducer, reducer_kind = ck.PeerAllreducer(params), "ck_allreduce_peers (CUDA IPC, fixed rank order)"
            except Exception as exc:  # IPC unavailable on this box: NCCL
                print(f"peer allreduce unavailable ({exc}); using NCCL", file=sys.stderr)
        if reducer is None:
            reducer, reducer_kind = ck.GradientAllreducer(params), "NCCL all_reduce (Ring)"
        # dC / db written by ck_backward straight into the exchange buffer; the
        # peer exchange starts on the grads-ready event, before the last dX GEMM
        reducer.bind(model)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    if is_net:
        # tabular / spectrogram-like features ~ N(0,1); regression target
        x = torch.randn(rows, I, device=dev, generator=gen)
        if O == 1:
            dy = torch.sin(x).sum(dim=1, keepdim=True) / 8 + 0.01 * torch.randn(rows, 1, device=dev, generator=gen)
        else:
            dy = torch.randn(rows, O, device=dev, generator=gen)
    else:
        x = (torch.rand(rows, I, device=dev, generator=gen) * 3.0 - 1.5).requires_grad_(True)
        dy = torch.randn(rows, O, device=dev, generator=gen)

    def step(xin, dyin, want_loss=False):
        """One training step; dyin is dL/dy (layer workloads) or the regression target (nets)."""
        if xin.requires_grad:
            xin.grad = None
        y = model(xin)
        if is_net:
            loss = ck.mse(y, dyin)
            loss.backward()
            loss = loss.detach() if want_loss else None
        else:
            loss = (y.detach() * dyin).sum() if want_loss else None  # L = sum(y * dy) -> dL/dy = dy
            y.backward(dyin)
        if reducer is not None:
            reducer()
        opt.step()
        opt.zero_grad(set_to_none=True)
        return loss

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local]) if backend == "nccl" else dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(ms):
        if world == 1:
            return ms
        t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    graph = None
    if use_graph:
        # whole-step CUDA graph (forward, backward, allreduce, Adam): the
        # small nets are launch-bound, so the step is captured once and
        # replayed; warm-up runs on a side stream as capture requires
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(args.warmup):
                step(x, dy)
        torch.cuda.current_stream(dev).wait_stream(side)
        barrier()
        graph = torch.cuda.CUDAGraph()
        launches_c0 = _lib.launch_count()
        with torch.cuda.graph(graph):
            step(x, dy)
        launches_per_step = _lib.launch_count() - launches_c0
        barrier()
    else:
        for _ in range(args.warmup):
            step(x, dy)
        barrier()

    def kernel_breakdown():
        """Per-class device time of eager steps (library event timers)."""
        _lib.timing_collect()
        _lib.timing_enable(True)
        for _ in range(args.steps):
            step(x, dy)
        barrier()
        _lib.timing_enable(False)
        return _lib.timing_collect()

    # ---- timed region: training steps, device-resident inputs -----------
    clocks = ClockSampler(local) if local == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    if graph is None:
        _lib.timing_collect()
        _lib.timing_enable(True)
    launches0 = _lib.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step(x, dy)
    ev1.record()
    barrier()
    if graph is None:
        launches = _lib.launch_count() - launches0
        _lib.timing_enable(False)
        kt = _lib.timing_collect()
    else:
        launches = launches_per_step * args.steps
    clk = clocks.stop() if clocks else None
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / args.steps
    value = gb / (ms_step / 1e3)
    if graph is not None:
        # replays advanced the parameters without Python seeing it: refresh the
        # version counters so the layers re-split their coefficients
        for prm in model.parameters():
            torch.autograd.graph.increment_version(prm)
        kt = kernel_breakdown()

    # ---- forward-only throughput (inference), same shard ---------------
    with torch.no_grad():
        xs = x.detach()
        for _ in range(2):
            model(xs)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            model(xs)
        f1.record()
        barrier()
        fwd_ms = max_over_ranks(f0.elapsed_time(f1)) / args.steps
    fwd_value = gb / (fwd_ms / 1e3)

    # ---- end to end: pinned host inputs streamed in, loss read back -----
    # The step's x / dy live in pinned host memory.  They are copied in
    # micro-batches of at most 32768 rows on a copy stream, double-buffered,
    # so the copy of micro-batch j+1 overlaps forward/backward of j; the
    # gradients accumulate across micro-batches (the usual data-loader /
    # gradient-accumulation pattern on the public module API), then one
    # allreduce + Adam step, then the loss is read back to the host.
    mb = min(rows, 32768)
    n_mb = (rows + mb - 1) // mb
    x_h = torch.empty((rows, I), dtype=torch.float32, pin_memory=True)
    dy_h = torch.empty((rows, O), dtype=torch.float32, pin_memory=True)
    x_h.copy_(x.detach())
    dy_h.copy_(dy)
    xb = [torch.empty((mb, I), device=dev) for _ in range(2)]
    dyb = [torch.empty((mb, O), device=dev) for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for ev in free:
        ev.record()

    pending = {"next": None}  # global micro-batch index already being copied

    def issue_copy(g):
        k, j = g & 1, g % n_mb
        lo, hi = j * mb, min(rows, (j + 1) * mb)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(free[k])
            xb[k][: hi - lo].copy_(x_h[lo:hi], non_blocking=True)
            dyb[k][: hi - lo].copy_(dy_h[lo:hi], non_blocking=True)
            ready[k].record(copy_stream)

    def e2e_step(step_no=0, prefetch_next_step=True):
        # continuous copy pipeline: the copy of micro-batch g+1 (possibly the
        # next step's first) is issued before the compute of g
        cur = torch.cuda.current_stream(dev)
        loss = torch.zeros((), device=dev)
        for j in range(n_mb):
            g = step_no * n_mb + j
            k = g & 1
            lo, hi = j * mb, min(rows, (j + 1) * mb)
            if pending["next"] != g:
                issue_copy(g)
            pending["next"] = None
            if j + 1 < n_mb or prefetch_next_step:
                issue_copy(g + 1)
                pending["next"] = g + 1
            cur.wait_event(ready[k])
            xin = xb[k][: hi - lo].detach().requires_grad_(not is_net)
            # micro-batches before the last accumulate without starting the exchange
            sync_ctx = reducer.no_sync() if (reducer is not None and j + 1 < n_mb) else contextlib.nullcontext()
            with sync_ctx:
                y = model(xin)
                if is_net:
                    part = ck.mse(y, dyb[k][: hi - lo]) * ((hi - lo) / rows)
                    part.backward()
                    loss += part.detach()
                else:
                    # L = sum(y * dy): one dot pass (mul + sum read the 0.5 GB twice)
                    loss += torch.dot(y.detach().reshape(-1), dyb[k][: hi - lo].reshape(-1))
                    y.backward(dyb[k][: hi - lo])
            free[k].record(cur)
        if reducer is not None:
            reducer()
        opt.step()
        opt.zero_grad(set_to_none=True)
        return float(loss.item())  # D2H of the step's result

    e2e_mode = (f"eager, {n_mb} micro-batches of {mb} rows; the copy of micro-batch g+1 (the next step's first "
                f"included) overlaps the compute of g")
    if graph is not None and n_mb == 1:
        # launch-bound nets: the e2e step's compute -- forward, backward, Adam,
        # D2H copy of the loss -- is one captured CUDA graph per input buffer;
        # the H2D copy of step s+1's x/dy (pinned memory, copy stream) runs
        # while step s computes, and every step's loss is read on the host
        loss_h = [torch.zeros((), dtype=torch.float32, pin_memory=True) for _ in range(2)]

        def e2e_body(k):
            y = model(xb[k][:rows])
            loss = ck.mse(y, dyb[k][:rows])
            loss.backward()
            opt.step()
            opt.zero_grad(set_to_none=True)
            loss_h[k].copy_(loss.detach(), non_blocking=True)

        for k in range(2):
            xb[k][:rows].copy_(x_h)
            dyb[k][:rows].copy_(dy_h)
        side2 = torch.cuda.Stream(device=dev)
        side2.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side2):
            for k in (0, 1, 0, 1):
                e2e_body(k)
        torch.cuda.current_stream(dev).wait_stream(side2)
        torch.cuda.synchronize(dev)
        barrier()
        g_e2e = []
        for k in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                e2e_body(k)
            g_e2e.append(g)
        torch.cuda.synchronize(dev)

        done = [torch.cuda.Event() for _ in range(2)]
        last = {"k": None}

        def e2e_step(step_no=0, prefetch_next_step=True):  # noqa: F811 (graph-replay form)
            # the host reads step s-1's loss (copied to pinned memory inside
            # its graph) after enqueueing step s, so the GPU never waits for
            # the host between steps; the last step of a run reads its own
            cur = torch.cuda.current_stream(dev)
            k = step_no & 1
            if pending["next"] != step_no:
                issue_copy(step_no)
            pending["next"] = None
            if prefetch_next_step:
                issue_copy(step_no + 1)  # overlaps this step's compute
                pending["next"] = step_no + 1
            cur.wait_event(ready[k])
            g_e2e[k].replay()
            free[k].record(cur)
            done[k].record(cur)
            out = None
            if last["k"] is not None:
                done[last["k"]].synchronize()
                out = float(loss_h[last["k"]])
            last["k"] = k
            if not prefetch_next_step:
                done[k].synchronize()
                out = float(loss_h[k])
                last["k"] = None
            return out

        e2e_mode = ("one captured CUDA graph per step (forward, backward, Adam, D2H copy of the loss); every "
                    "step's loss is read on the host one step later (after the next step is enqueued) and the "
                    "H2D copy of the next step's x/dy from pinned memory overlaps this step's compute")
    e2e_step(0, prefetch_next_step=False)  # warm the copy path; no copy left in flight
    barrier()
    e2e_steps = max(10, args.steps)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for si in range(e2e_steps):
        e2e_step(si, prefetch_next_step=si + 1 < e2e_steps)
    e1.record()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
    e2e_wall = (time.perf_counter() - t0) / e2e_steps
    e2e_value = gb / (e2e_ms / 1e3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    # Executed GEMM flops (SURVEY 8(d) with the B_0 == 1 folds subtracted):
    # forward and dC contract over d planes (k = 1..d), dX over d planes; a
    # net's first layer has no dX (its input needs no gradient).  The
    # algorithmic 8(d) count 2*B*I*O*(3d+2) (k = 0 included) is reported beside.
    train_alg, step_gemm, fwd_gemm = 0, 0, 0
    for li, (i, o) in enumerate(dims):
        need_dx = not (is_net and li == 0)
        train_alg += 2 * rows * i * o * ((d + 1) + (d + 1) + (d if need_dx else 0))
        step_gemm += 2 * rows * i * o * d * (3 if need_dx else 2)
        fwd_gemm += 2 * rows * i * o * d
    gemm_alg = step_gemm * args.steps
    gemm_ms = sum(kt[c][0] for c in ("gemm_fwd", "gemm_dx", "gemm_dc"))
    gemm_tf = gemm_alg / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    # Denominator: the measured bf16 BURST figure / 3.  The kernel runs inside a
    # long power-capped step, but the box-to-box clock under the 1 kW cap
    # varies (1.1-1.35 GHz seen), so the pod's sustained figure (cuBLAS at the
    # measuring pod's capped clock) can sit below what a cooler box reaches;
    # the burst figure keeps frac <= 1 and is the conservative choice.
    peak_eff = peaks["bf16"] / 3.0
    total_kernel_ms = sum(v[0] for v in kt.values())
    # DRAM bytes per GEMM launch from the committed ncu --set full capture of
    # this exact launch (C4, 32768-row chunk); other workloads: not measured
    traffic, traffic_src = None, None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists() and not is_net and (I, O, d) == (4096, 4096, 8):
        try:
            tj = json.loads(tp.read_text())
            traffic, traffic_src = tj.get("gemm_bf16x3_bytes_per_launch"), tj.get("source")
        except (ValueError, OSError):
            traffic = None
    line = {
        "metric": METRIC_NET if is_net else METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if wl.get("weak") else "strong", "vs_baseline": None,
        "dtype": "fp32 I/O, bf16x3 split tensor-core products, fp32 accumulate", "data": "synthetic",
        "config": {"workload": wl["name"], "global_batch": gb, "rows_per_gpu": rows, "layers": dims,
                   "degree": d, "lut_size": wl["lut_size"], "parallelism": f"dp{world}",
                   "gradient_exchange": reducer_kind,
                   "l2": ("inputs larger than L2 (x shard >> 126 MB), no flush" if rows * I * 4 > 126e6 else
                          "working set below L2 size; steps run back to back (no flush)")},
        "fwd": {"value": fwd_value, "unit": "samples/s", "ms_per_step": fwd_ms,
                "tflops_executed": fwd_gemm / (fwd_ms / 1e3) / 1e12,
                "roofline_frac": fwd_gemm / (fwd_ms / 1e3) / 1e12 / peak_eff,
                "roofline_basis": "whole forward time (expansion + GEMM) vs bf16 burst / 3"},
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": 4 * rows * (I + O),
                "d2h_bytes_per_step": 4, "ms_per_step": e2e_ms, "wall_ms_per_step": e2e_wall * 1e3,
                "path": f"ChebyKANLayer forward/backward + Adam; x/dy from pinned host: {e2e_mode}"},
        "gpu_launches": launches,
        "roofline": {
            "bound": "tensor", "kernel": "gemm_bf16x3 (tcgen05 fwd + dX + dC, BF16x3)",
            "achieved": gemm_tf, "peak": peak_eff, "unit": "TFLOP/s", "frac": gemm_tf / peak_eff,
            "traffic": traffic, "traffic_source": traffic_src,
            "peak_basis": f"{peaks['source']} bf16 burst {peaks['bf16']} TF/s / 3 (3 bf16 MMAs per "
                          f"algorithmic fp32 MMA); sustained {peaks['bf16_sus']} TF/s gives frac "
                          f"{gemm_tf / (peaks['bf16_sus'] / 3.0):.3f}",
            "algorithmic_flops_per_step": step_gemm,
            "gemm_share_of_kernel_time": gemm_ms / total_kernel_ms if total_kernel_ms else None,
            # the part is power-capped: the same achieved rate against the
            # tensor pipe's per-clock peak (148 SMs x 8192 dense bf16 flop/clk,
            # / 3 for BF16x3) at the SM clock sampled during the timed region
            "frac_at_sampled_clock": (gemm_tf / (148 * 8192 * clk["sm_mhz"] * 1e6 / 3 / 1e12)
                                      if clk and clk.get("sm_mhz") else None),
        },
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items() if v[1]},
        "graph": (f"timed steps replay one captured CUDA graph of the whole step; kernel_ms_per_step and "
                  f"roofline from {args.steps} eager steps" if graph is not None else None),
        "kernel_launches_per_step": {k: v[1] / args.steps for k, v in kt.items() if v[1]},
        "train_tflops_per_gpu": {"executed": step_gemm / (ms_step / 1e3) / 1e12,
                                 "algorithmic_8d": train_alg / (ms_step / 1e3) / 1e12,
                                 "note": "executed = k >= 1 planes only (the B_0 == 1 folds are not work done)"},
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        base, cpu_layers, cpu_outs = cpu_baseline(wl, CPU_SAMPLE_ROWS)
        line["cpu_baseline"] = base
        line["parity"] = gpu_parity(wl, cpu_layers, cpu_outs)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sweep(args):
    """C1 sweep: I=O in 256..4096 x degree in {3,4,5,8}, batch 16384, fwd and fwd+bwd (1 GPU)."""
    import torch

    import paper_2511_14852_b200 as ck
    from paper_2511_14852_b200.kernels import PreparedCoeff, backward_raw, forward_raw

    dev = torch.device("cuda", 0)
    peaks = load_peaks()
    rows = []
    for dim in (256, 512, 1024, 2048, 4096):
        for deg in (3, 4, 5, 8):
            b = 16384
            x = torch.rand(b, dim, device=dev) * 3 - 1.5
            c = (torch.rand(deg + 1, dim, dim, device=dev) * 2 - 1) / (dim * (deg + 1)) ** 0.5
            dy = torch.randn(b, dim, device=dev)
            lut = ck.lut_build(ck.BasisKind.CHEBYSHEV, deg, 32768, device=dev)
            prep = PreparedCoeff(c)
            cache = torch.empty(ck.kernels.basis_cache_bytes(b, dim, dim, deg + 1), dtype=torch.uint8, device=dev)

            def infer():
                forward_raw(x, prep, lut, None)

            def train():
                forward_raw(x, prep, lut, None, cache)
                backward_raw(x, dy, prep, lut, True, cache=cache)

            for _ in range(3):
                infer()
                train()
            torch.cuda.synchronize()
            if args.graph is not False:
                # the small layers are launch-bound: time captured CUDA graphs
                graphs = []
                for fn in (infer, train):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        fn()
                    graphs.append(g.replay)
                infer_run, train_run = graphs
            else:
                infer_run, train_run = infer, train
            for _ in range(2):
                infer_run()
                train_run()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            for _ in range(args.steps):
                infer_run()
            ev[1].record()
            for _ in range(args.steps):
                train_run()
            ev[2].record()
            torch.cuda.synchronize()
            f = ev[0].elapsed_time(ev[1]) / args.steps
            bw = ev[1].elapsed_time(ev[2]) / args.steps - f
            fl = ck.count_flops(b, dim, dim, deg)
            # executed GEMM flops: the T_0 == 1 folds remove one of the d+1
            # planes from the forward and dC GEMMs
            ex_f = 2 * b * dim * dim * deg
            ex_t = 3 * ex_f
            peak = peaks["bf16"] / 3.0
            r = {"d_in": dim, "d_out": dim, "degree": deg, "batch": b, "fwd_ms": f, "bwd_ms": bw,
                 "fwd_samples_per_s": b / f * 1e3, "train_samples_per_s": b / (f + bw) * 1e3,
                 "fwd_alg_tflops": fl["fwd"] / f / 1e9, "train_alg_tflops": fl["train"] / (f + bw) / 1e9,
                 "fwd_exec_tflops": ex_f / f / 1e9, "train_exec_tflops": ex_t / (f + bw) / 1e9,
                 "fwd_frac_of_bf16x3_burst": ex_f / f / 1e9 / peak,
                 "train_frac_of_bf16x3_burst": ex_t / (f + bw) / 1e9 / peak}
            rows.append(r)
            print(json.dumps(r), flush=True)
            del x, c, dy, prep, cache
    out = ROOT / "gpurun_out" / "sweep.json"
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(rows, indent=1))


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--sweep", action="store_true", help="run the C1 sweep table instead of the JSON line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reducer", choices=("peer", "nccl"), default="peer",
                    help="N>1 gradient exchange: the library's peer-memory kernel or NCCL")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="replay a captured CUDA graph of the step (default for the small nets)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours" and not args.sweep:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
    elif args.sweep:
        run_sweep(args)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
