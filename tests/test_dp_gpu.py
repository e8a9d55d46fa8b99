"""Data-parallel numerics on the GPU: two ranks (gloo, both on cuda:0 -- this
sandbox has one device and NCCL refuses two ranks per GPU) each run the fused
layer on their contiguous shard and allreduce [dC, db]; the reduced gradients
must equal the single-process full-batch gradients."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grads(layer, x, dy):
    layer.zero_grad(set_to_none=True)
    xx = x.clone().requires_grad_(True)
    layer(xx).backward(dy)
    return layer.coeff_doj.grad.clone(), layer.bias.grad.clone(), xx.grad.clone()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_14852_b200 as ck

    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    layer = ck.ChebyKANLayer(96, 80, 5, lut_size=4096, seed=3).to(dev)
    g = torch.Generator().manual_seed(7)
    B = 1000
    x = (torch.rand(B, 96, generator=g) * 3 - 1.5).to(dev)
    dy = torch.randn(B, 80, generator=g).to(dev)
    lo, hi = ck.shard_bounds(B, rank, world)
    dc, db, dx = _grads(layer, x[lo:hi], dy[lo:hi])
    red = ck.GradientAllreducer(ck.chebykan_parameters(layer))
    red()
    q.put((rank, layer.coeff_doj.grad.cpu().numpy(), layer.bias.grad.cpu().numpy(), dx.cpu().numpy(), lo, hi))
    dist.destroy_process_group()


def test_dp_two_ranks_match_full_batch():
    import paper_2511_14852_b200 as ck
    from oracle import chebykan_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    layer = ck.ChebyKANLayer(96, 80, 5, lut_size=4096, seed=3).to(dev)
    g = torch.Generator().manual_seed(7)
    x = (torch.rand(1000, 96, generator=g) * 3 - 1.5).to(dev)
    dy = torch.randn(1000, 80, generator=g).to(dev)
    dc, db, dx = _grads(layer, x, dy)
    for r in (0, 1):
        rdc, rdb, rdx, lo, hi = res[r]
        assert orc.normwise_err(rdc, dc.cpu().numpy()) <= 1e-5
        assert orc.normwise_err(rdb, db.cpu().numpy()) <= 1e-6
        assert orc.normwise_err(rdx, dx[lo:hi].cpu().numpy()) <= 1e-6
    assert np.array_equal(res[0][0], res[1][0])  # identical reduced gradients on both ranks


def _peer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_14852_b200 as ck

    dev = torch.device("cuda", 0)
    net = torch.nn.Sequential(ck.ChebyKANLayer(64, 48, 4, lut_size=2048, seed=1),
                              ck.ChebyKANLayer(48, 5, 3, lut_size=2048, seed=2)).to(dev)
    params = ck.chebykan_parameters(net)
    g = torch.Generator().manual_seed(100 + rank)
    for p in params:  # rank-specific gradients standing in for ck_backward's
        p.grad = torch.randn(p.shape, generator=g).to(dev)
    local = [p.grad.clone().cpu() for p in params]
    red = ck.PeerAllreducer(params)
    for _ in range(2):  # reusable: second call on fresh copies gives the same bits
        for p, l in zip(params, local):
            p.grad.copy_(l.to(dev))
        red()
    q.put((rank, [l.numpy() for l in local], [p.grad.cpu().numpy() for p in params]))
    red.close()
    dist.destroy_process_group()


def test_peer_allreduce_fixed_order_bitwise():
    # ck_allreduce_peers over CUDA IPC (two processes on one device): the sum
    # is rank 0 + rank 1 in that order, bit-identical on both ranks
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i in range(len(res[0][0])):
        want = (res[0][0][i].astype(np.float32) + res[1][0][i].astype(np.float32)).astype(np.float32)
        assert np.array_equal(res[0][1][i], want)
        assert np.array_equal(res[1][1][i], want)


def _bound_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_14852_b200 as ck

    dev = torch.device("cuda", 0)
    net = torch.nn.Sequential(ck.ChebyKANLayer(64, 48, 4, lut_size=2048, seed=1),
                              ck.ChebyKANLayer(48, 5, 3, lut_size=2048, seed=2)).to(dev)
    red = ck.PeerAllreducer(ck.chebykan_parameters(net)).bind(net)
    g = torch.Generator().manual_seed(9)
    B = 600
    x = (torch.rand(B, 64, generator=g) * 3 - 1.5).to(dev)
    dy = torch.randn(B, 5, generator=g).to(dev)
    lo, hi = ck.shard_bounds(B, rank, world)
    outs = []
    for _ in range(2):  # the same step twice: bit-identical
        net.zero_grad(set_to_none=True)
        net(x[lo:hi]).backward(dy[lo:hi])
        red()
        torch.cuda.synchronize()
        grads = [p.grad.detach().clone().cpu().numpy() for p in red.params]
        inplace = [p.grad.data_ptr() == v.data_ptr() for p, v in zip(red.params, red.views)]
        outs.append((grads, inplace))
    q.put((rank, outs))
    red.close()
    dist.destroy_process_group()


def test_peer_allreduce_bound_inplace_matches_full_batch():
    """bind(): the backward writes dC / db into the exchange buffer, each
    layer's exchange runs on a side stream behind ck_backward's grads-ready
    event (device flags, no host barrier); the summed gradients equal the
    full-batch ones, bit-identical on both ranks and run to run."""
    import paper_2511_14852_b200 as ck
    from oracle import chebykan_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_bound_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    net = torch.nn.Sequential(ck.ChebyKANLayer(64, 48, 4, lut_size=2048, seed=1),
                              ck.ChebyKANLayer(48, 5, 3, lut_size=2048, seed=2)).to(dev)
    g = torch.Generator().manual_seed(9)
    x = (torch.rand(600, 64, generator=g) * 3 - 1.5).to(dev)
    dy = torch.randn(600, 5, generator=g).to(dev)
    net(x).backward(dy)
    want = [p.grad.cpu().numpy() for p in ck.chebykan_parameters(net)]
    for r in (0, 1):
        for grads, inplace in res[r]:
            assert all(inplace), inplace
            for gg, w in zip(grads, want):
                assert orc.normwise_err(gg, w) <= 1e-5
    for (g0, _), (g1, _) in zip(res[0], res[1]):
        for a, b in zip(g0, g1):
            assert np.array_equal(a, b)
    for a, b in zip(res[0][0][0], res[0][1][0]):
        assert np.array_equal(a, b)


def _nccl_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import paper_2511_14852_b200 as ck

    ck.parallel.deterministic_nccl_env()
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    net = ck.ChebyKANLayer(96, 80, 5, lut_size=4096, seed=3).to(dev)
    red = ck.GradientAllreducer(ck.chebykan_parameters(net)).bind(net)
    g = torch.Generator().manual_seed(11 + rank)
    x = (torch.rand(300, 96, generator=g) * 3 - 1.5).to(dev)
    dy = torch.randn(300, 80, generator=g).to(dev)
    runs = []
    for _ in range(3):
        net.zero_grad(set_to_none=True)
        net(x).backward(dy)
        red()
        runs.append([p.grad.cpu().numpy().copy() for p in red.params])
    q.put((rank, runs))
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="NCCL needs one GPU per rank")
def test_nccl_allreduce_bitwise_run_to_run():
    """GradientAllreducer over NCCL (Ring / Simple pinned): the same step three
    times gives bit-identical summed gradients, equal on both ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        for run in res[r][1:]:
            for a, b in zip(res[r][0], run):
                assert np.array_equal(a, b)
    for a, b in zip(res[0][0], res[1][0]):
        assert np.array_equal(a, b)
