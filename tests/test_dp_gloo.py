"""World-size-2 data-parallel plumbing on CPU (gloo): batch sharding plus one
flat allreduce of the ChebyKAN coefficient/bias gradients."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_14852_b200 import ChebyKANLayer, GradientAllreducer, chebykan_parameters, shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        net = torch.nn.Sequential(ChebyKANLayer(6, 5, 3, seed=1), ChebyKANLayer(5, 2, 2, seed=2))
        params = chebykan_parameters(net)
        assert len(params) == 4
        # deterministic per-rank fake gradients standing in for ck_backward's
        gb = 10
        a, b = shard_bounds(gb, rank, world)
        for i, p in enumerate(params):
            g = torch.arange(p.numel(), dtype=torch.float32).reshape(p.shape) * (i + 1)
            p.grad = g * (b - a)  # proportional to the rows this rank owns
        red = GradientAllreducer(params)
        # one flat buffer, every slot 16-byte aligned
        assert red.nbytes == 4 * sum((p.numel() + 3) // 4 * 4 for p in params)
        red()
        out_q.put((rank, [p.grad.clone().numpy() for p in params]))
    finally:
        dist.destroy_process_group()


def test_gradient_allreduce_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank holds the sum over ranks: sum_r rows_r * base = 10 * base
    for r in range(world):
        for i, g in enumerate(results[r]):
            base = np.arange(g.size, dtype=np.float32).reshape(g.shape) * (i + 1)
            np.testing.assert_array_equal(g, base * 10)
    for g0, g1 in zip(results[0], results[1]):
        np.testing.assert_array_equal(g0, g1)
