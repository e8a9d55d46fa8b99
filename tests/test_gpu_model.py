"""Model / trainer layer on the GPU vs the reference trainer's trajectories.

Fixtures: tests/golden/train_*.npz from tests/golden/make_golden_train.py
(the reference's network_train, model.py:380-460).  The GPU trainer runs in
float32 with BF16x3 tensor-core contractions, the reference in float64, so
trajectories agree to round-off amplified over a few dozen Adam steps:
epoch losses within 1e-3 relative, final parameters within 1e-3 normwise.
"""
import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import chebykan_oracle as orc

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2511_14852_b200 as ck

TRAIN_TOL = 1e-3


def _cases():
    K = ck.BasisKind
    exact = ck.KernelMode(ck.BasisPath.EXACT_RECURRENCE)
    # mirrors CASES in tests/golden/make_golden_train.py
    return {
        "cheb2": ((ck.LayerSpec(1, 8, 4), ck.LayerSpec(8, 1, 4)), ck.Loss.MSE, 3, 4096, 0, 1e-2, 32, True),
        "sincos_mixed": ((ck.LayerSpec(2, 6, 3, K.LEGENDRE), ck.LayerSpec(6, 1, 3, mode=exact)), ck.Loss.MSE, 3,
                         2048, 3, 5e-3, 32, True),
        "sectors_ce": ((ck.LayerSpec(2, 5, 3), ck.LayerSpec(5, 3, 2, K.FOURIER)), ck.Loss.CROSS_ENTROPY, 3, 4096,
                       5, 1e-2, 16, False),
        "positive_rmsle": ((ck.LayerSpec(3, 4, 2, K.HERMITE), ck.LayerSpec(4, 1, 2, has_bias=False)),
                           ck.Loss.RMSLE, 2, 1024, 9, 1e-2, 20, True),
    }


@pytest.mark.parametrize("name", ["cheb2", "sincos_mixed", "sectors_ce", "positive_rmsle"])
def test_network_train_follows_reference_trajectory(name):
    g = np.load(GOLDEN / f"train_{name}.npz")
    layers, loss, epochs, lut_size, seed, lr, batch, cosine = _cases()[name]
    ds = ck.Dataset(g["x"], g["y"], name=name)
    res = ck.network_train(ck.NetworkSpec(layers, loss), ds, epochs, ck.AdamHParams(lr=lr), seed=seed,
                           batch_size=batch, lut_size=lut_size, cosine_decay=cosine)
    got = np.array(res.trace.epoch_losses)
    want = g["epoch_losses"]
    print(name, got, want)
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= TRAIN_TOL * np.abs(want).max()
    for i, layer in enumerate(res.network.layers):
        c = layer.coeff.as3d().permute(2, 1, 0).cpu().numpy()
        assert orc.normwise_err(c, g[f"coeff_jod_{i}"]) <= TRAIN_TOL
        if layer.bias is not None:
            assert np.abs(layer.bias.cpu().numpy() - g[f"bias_{i}"]).max() <= TRAIN_TOL * max(
                1.0, np.abs(g[f"bias_{i}"]).max())
    assert len(res.trace.fwd_seconds) == epochs and all(t > 0 for t in res.trace.fwd_seconds)


def test_init_params_bit_identical_to_reference_draws():
    spec = ck.LayerSpec(7, 5, 3)
    coeff, bias = ck.init_params(spec, seed=11)
    rng = np.random.default_rng(11)
    s = 1.0 / np.sqrt(7 * 4)
    assert np.array_equal(coeff.data.numpy().reshape(-1), rng.uniform(-s, s, size=7 * 5 * 4))
    assert np.array_equal(bias.numpy(), np.zeros(5))


def test_layer_api_backward_before_forward_and_shapes():
    layer = ck.Layer.create(ck.LayerSpec(4, 3, 2), seed=0, lut_size=256)
    with pytest.raises(RuntimeError, match="backward called before forward"):
        layer.backward(np.zeros((2, 3)))
    with pytest.raises(ValueError, match=r"expected input shape \(batch, 4\)"):
        layer.forward(np.zeros((2, 5)))
    x = np.random.default_rng(0).uniform(-1, 1, (6, 4))
    y = layer.forward(x)
    cg, bg, xg = layer.backward(np.ones((6, 3)))
    assert tuple(y.shape) == (6, 3) and tuple(xg.shape) == (6, 4)
    assert cg.layout is ck.Layout.DOJ and tuple(cg.data.shape) == (3, 3, 4)
    assert torch.allclose(bg, torch.full((3,), 6.0, device=bg.device))


def test_adam_kernel_matches_reference_rule():
    # model.py:247-266 on float64 vs ck_adam_step on float32, three steps
    rng = np.random.default_rng(3)
    p0 = rng.standard_normal(1001)
    grads = [rng.standard_normal(1001) for _ in range(3)]
    p, m, v = p0.copy(), np.zeros(1001), np.zeros(1001)
    lr, b1, b2, eps = 1e-2, 0.9, 0.999, 1e-8
    for t, gr in enumerate(grads, start=1):
        m = m * b1 + (1 - b1) * gr
        v = v * b2 + (1 - b2) * (gr * gr)
        p = p - lr * (m / (1 - b1 ** t)) / (np.sqrt(v / (1 - b2 ** t)) + eps)
    dev = torch.device("cuda", 0)
    pt = torch.tensor(p0, dtype=torch.float32, device=dev)
    mt, vt = torch.zeros_like(pt), torch.zeros_like(pt)
    for t, gr in enumerate(grads, start=1):
        ck.adam_update(pt, torch.tensor(gr, dtype=torch.float32, device=dev), mt, vt, lr, b1, b2, eps, t)
    assert np.abs(pt.cpu().numpy() - p).max() <= 1e-6


@pytest.mark.parametrize("capturable", [False, True])
def test_multi_tensor_adam_bitwise_equals_per_tensor(capturable):
    # ck_adam_step_multi (one launch, 40 tensors -> two launches of <= 32, ragged
    # sizes with tails that are not whole float4s) == ck_adam_step per tensor, bit for bit.
    # Zero-size tensors inside the first batch must not shift the batch
    # boundary (each tensor updated exactly once).
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(5)
    sizes = [1, 0, 3, 2047, 0, 2048, 2049, 4096 + 5, 17, 100000] + [
        int(s) for s in torch.randint(1, 5000, (32,), generator=g)]
    params = [torch.nn.Parameter(torch.randn(n, generator=g).to(dev)) for n in sizes]
    ref = [p.detach().clone() for p in params]
    ms = [torch.zeros_like(p) for p in ref]
    vs = [torch.zeros_like(p) for p in ref]
    opt = ck.Adam(params, lr=3e-3, capturable=capturable)
    for t in range(1, 4):
        grads = [torch.randn(n, generator=g).to(dev) for n in sizes]
        for p, gr in zip(params, grads):
            p.grad = gr.clone()
        opt.step()
        for r, gr, m, v in zip(ref, grads, ms, vs):
            ck.adam_update(r, gr, m, v, 3e-3, 0.9, 0.999, 1e-8, t)
    for p, r in zip(params, ref):
        assert torch.equal(p.detach(), r)


def test_training_divergence_reports_epoch_and_batch():
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (64, 2))
    y = np.full(64, np.inf)
    spec = ck.NetworkSpec((ck.LayerSpec(2, 3, 2), ck.LayerSpec(3, 1, 2)))
    with pytest.raises(ck.TrainingDiverged, match="epoch 0, batch 0"):
        ck.network_train(spec, ck.Dataset(x, y), 1, lut_size=256)


def test_cuda_graph_training_step_matches_eager():
    # whole-step capture (forward, backward, capturable Adam) replayed N times
    # must follow the eager trajectory (device-side Adam step counter)
    dev = torch.device("cuda", 0)

    def make():
        torch.manual_seed(0)
        m = torch.nn.Sequential(ck.ChebyKANLayer(24, 40, 4, lut_size=2048), ck.ChebyKANLayer(40, 3, 3, lut_size=2048),
                                ).to(dev)
        return m

    x = torch.randn(512, 24, device=dev)
    tgt = torch.randn(512, 3, device=dev)

    def run(model, opt):
        loss = torch.nn.functional.mse_loss(model(x), tgt)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)

    eager = make()
    opt_e = ck.Adam(eager.parameters(), lr=1e-2)
    for _ in range(7):
        run(eager, opt_e)

    graphed = make()
    opt_g = ck.Adam(graphed.parameters(), lr=1e-2, capturable=True)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            run(graphed, opt_g)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run(graphed, opt_g)
    for _ in range(4):
        g.replay()
    torch.cuda.synchronize()
    # 3 warm-up + 4 replays = 7 updates (capture records, it does not execute)
    for pe, pg in zip(eager.parameters(), graphed.parameters()):
        assert torch.allclose(pe, pg, rtol=1e-5, atol=1e-6), (pe - pg).abs().max()


def _net_cases():
    # mirrors NET_CASES in tests/golden/make_golden_train.py (BASELINE configs C2 / C3 at full width)
    return {
        "c2_tabular": ((ck.LayerSpec(64, 512, 5), ck.LayerSpec(512, 512, 5), ck.LayerSpec(512, 1, 5)), 2, 32768, 1,
                       1e-4, 64, 1e-3),
        "c3_speech": ((ck.LayerSpec(257, 512, 15), ck.LayerSpec(512, 512, 15), ck.LayerSpec(512, 257, 15)), 2, 32768,
                      2, 3e-5, 64, 2e-3),
    }


@pytest.mark.parametrize("name", ["c2_tabular", "c3_speech"])
def test_c2_c3_nets_follow_reference_trajectory(name):
    """network_train on the C2 tabular net [64->512->512->1] d5 and the C3
    speech FFN [257->512->512->257] d15 (256 rows, 2 epochs of 4 Adam steps,
    cosine decay) against the reference trainer's float64 run.

    Bars: epoch losses within 1e-3 relative; the
    trained network's outputs on a probe batch within 1e-3 (C2) / 2e-3 (C3)
    normwise -- the reference's own outputs move by 1.1e-4 / 5.8e-4 when
    1e-5 * max|g| of additive noise (the size of a BF16x3 gradient error)
    perturbs its gradients (tests/golden/make_golden_train.py).  The
    coefficients (a fixed-stride subsample) are compared elementwise at
    1e-3 of their range for all but <= 0.1 % of the elements, the biases
    (which start at 0, so their range is only ~lr * steps) to 1 % of their
    range: Adam's first
    step is ~lr * sign(g), so an element whose gradient lies below the
    round-off can take the opposite first step -- a discrete difference of
    2 lr, not a drift."""
    g = np.load(GOLDEN / f"train_{name}.npz")
    layers, epochs, lut_size, seed, lr, batch, probe_tol = _net_cases()[name]
    ds = ck.Dataset(g["x"].astype(np.float64), g["y"].astype(np.float64), name=name)
    res = ck.network_train(ck.NetworkSpec(layers, ck.Loss.MSE), ds, epochs, ck.AdamHParams(lr=lr), seed=seed,
                           batch_size=batch, lut_size=lut_size, cosine_decay=True)
    got = np.array(res.trace.epoch_losses)
    want = g["epoch_losses"]
    loss_err = float(np.abs(got - want).max() / np.abs(want).max())
    probe = res.network.forward(g["x"][: g["probe_y"].shape[0]].astype(np.float64))
    probe_err = orc.normwise_err(probe.cpu().numpy(), g["probe_y"])
    print(name, "losses", got, want, f"rel {loss_err:.2e}", f"probe {probe_err:.2e}")
    assert loss_err <= TRAIN_TOL
    assert probe_err <= probe_tol
    for i, layer in enumerate(res.network.layers):
        c = layer.coeff.as3d().permute(2, 1, 0).contiguous().cpu().numpy()
        assert tuple(c.shape) == tuple(g[f"coeff_jod_shape_{i}"])
        sub = c.reshape(-1)[::997]
        want_sub = g[f"coeff_jod_sub_{i}"]
        scale = np.abs(want_sub).max()
        bad = np.abs(sub - want_sub) > TRAIN_TOL * scale
        print(f"  layer {i}: coeff subsample normwise {orc.normwise_err(sub, want_sub):.2e}, "
              f"{int(bad.sum())}/{bad.size} beyond 1e-3")
        assert bad.mean() <= 1e-3
        if layer.bias is not None:
            # biases start at 0 and only move by Adam steps (~lr each), so their
            # range is ~lr * steps and gradients near Adam's eps make the
            # update proportional to the gradient's round-off: 1 % of the range
            gb, wb = layer.bias.cpu().numpy(), g[f"bias_{i}"]
            print(f"  layer {i}: bias normwise {orc.normwise_err(gb, wb):.2e}")
            assert orc.normwise_err(gb, wb) <= 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 4096, 1 << 20])
def test_fused_mse_matches_float64_and_is_deterministic(n):
    # ck_mse_loss: loss = mean((p - t)^2), grad = 2 (p - t) / n (model.py:184-218)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(n)
    p = torch.randn(n, generator=g).to(dev)
    t = torch.randn(n, generator=g).to(dev)
    loss, grad = ck.model.mse_device(p, t)
    pd, td = p.double().cpu().numpy(), t.double().cpu().numpy()
    want = np.mean((pd - td) ** 2)
    assert abs(float(loss) - want) <= 1e-6 * want
    np.testing.assert_allclose(grad.cpu().numpy(), 2.0 * (pd - td) / n, rtol=2e-7, atol=1e-12)
    again, _ = ck.model.mse_device(p, t)
    assert float(again) == float(loss)  # fixed-order reduction


@pytest.mark.gpu
def test_fused_mse_autograd_matches_torch():
    dev = torch.device("cuda", 0)
    torch.manual_seed(3)
    y = torch.randn(333, 5, device=dev, requires_grad=True)
    tgt = torch.randn(333, 5, device=dev, requires_grad=True)
    (3.0 * ck.mse(y, tgt)).backward()
    gy, gt = y.grad.clone(), tgt.grad.clone()
    y.grad, tgt.grad = None, None
    (3.0 * torch.nn.functional.mse_loss(y, tgt)).backward()
    torch.testing.assert_close(gy, y.grad, rtol=1e-6, atol=1e-9)
    torch.testing.assert_close(gt, tgt.grad, rtol=1e-6, atol=1e-9)
