"""Training-trajectory fixtures from the REFERENCE trainer (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_train.py

Runs polykan.model.network_train (model.py:380-460) -- seeded init, seeded
shuffles, Adam with cosine decay -- on the reference's synthetic datasets
and on small classification / RMSLE sets, and stores the per-epoch losses,
the final JOD coefficients and biases in tests/golden/train_*.npz.  The
GPU trainer (paper_2511_14852_b200.model.network_train) must follow the
same trajectory within float32 round-off.
"""
from __future__ import annotations

import pathlib

import numpy as np

from polykan.basis import BasisKind
from polykan.kernels import BasisPath, KernelMode
from polykan.model import (AdamHParams, Dataset, LayerSpec, Loss, NetworkSpec, make_synthetic, network_train)
from polykan.tensor import reorder_to_jod

HERE = pathlib.Path(__file__).resolve().parent
EXACT = KernelMode(BasisPath.EXACT_RECURRENCE)


def classification_set():
    rng = np.random.default_rng(7)
    x = rng.uniform(-1.5, 1.5, size=(96, 2))
    y = (np.floor((np.arctan2(x[:, 1], x[:, 0]) + np.pi) / (2 * np.pi / 3)) % 3).astype(np.int64)
    return Dataset(x, y, name="sectors")


def rmsle_set():
    rng = np.random.default_rng(8)
    x = rng.uniform(-1.0, 1.0, size=(80, 3))
    y = np.exp(0.5 * x[:, 0] + 0.25 * x[:, 1] ** 2) - 0.5 + 0.1 * x[:, 2]
    return Dataset(x, np.maximum(y, 0.0), name="positive")


CASES = [
    # name, dataset, layer specs, loss, epochs, lut_size, seed, lr, batch, cosine
    ("cheb2", make_synthetic("cheb2"), (LayerSpec(1, 8, 4), LayerSpec(8, 1, 4)), Loss.MSE, 3, 4096, 0, 1e-2, 32,
     True),
    ("sincos_mixed", make_synthetic("sincos"),
     (LayerSpec(2, 6, 3, BasisKind.LEGENDRE), LayerSpec(6, 1, 3, mode=EXACT)), Loss.MSE, 3, 2048, 3, 5e-3, 32, True),
    ("sectors_ce", classification_set(), (LayerSpec(2, 5, 3), LayerSpec(5, 3, 2, BasisKind.FOURIER)),
     Loss.CROSS_ENTROPY, 3, 4096, 5, 1e-2, 16, False),
    ("positive_rmsle", rmsle_set(), (LayerSpec(3, 4, 2, BasisKind.HERMITE), LayerSpec(4, 1, 2, has_bias=False)),
     Loss.RMSLE, 2, 1024, 9, 1e-2, 20, True),
]


def tabular_set():
    """C2 tabular regression: 64 features ~ N(0,1), target
    sum_j sin(x_j) / 8 + 0.01 noise; float32-representable values."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((256, 64)).astype(np.float32).astype(np.float64)
    y = (np.sin(x).sum(axis=1) / 8 + 0.01 * rng.standard_normal(256)).astype(np.float32).astype(np.float64)
    return Dataset(x, y, name="tabular")


def speech_set():
    """C3 speech enhancement (FFN replacement): 257 log-magnitude-like bins
    ~ N(0,1) per frame, target = a smooth per-bin map of the noisy frame."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((256, 257)).astype(np.float32).astype(np.float64)
    y = (0.5 * np.tanh(x) + 0.1 * np.roll(x, 1, axis=1)).astype(np.float32).astype(np.float64)
    return Dataset(x, y, name="speech")


# The BASELINE.json model configs C2 / C3 at full width on a 256-row set,
# 2 epochs of 4 batches.  Learning rates are chosen where the trajectory is
# well conditioned: at lr = 1e-3 the reference itself moves its final
# network by 1e-2 (C2) / 0.9 (C3) when 1e-5 * max|g| of additive noise -- the
# size of a float32 / BF16x3 gradient error -- is added to its gradients
# (Adam's first step is ~lr * sign(g), so near-zero gradients flip).  At the
# rates below the same perturbation moves the probe outputs by 1.1e-4 (C2)
# and 5.8e-4 (C3) and the epoch losses by <= 1.5e-5.  Their coefficients are large (8.4 M for C3), so
# the fixtures keep the epoch losses, the final network's outputs on a probe
# batch, the biases and a fixed-stride subsample of the JOD coefficients.
NET_CASES = [
    ("c2_tabular", tabular_set(), (LayerSpec(64, 512, 5), LayerSpec(512, 512, 5), LayerSpec(512, 1, 5)), Loss.MSE,
     2, 32768, 1, 1e-4, 64, True),
    ("c3_speech", speech_set(), (LayerSpec(257, 512, 15), LayerSpec(512, 512, 15), LayerSpec(512, 257, 15)),
     Loss.MSE, 2, 32768, 2, 3e-5, 64, True),
]
SUBSAMPLE_STRIDE = 997
PROBE_ROWS = 64


def main_nets():
    for name, ds, layers, loss, epochs, lut_size, seed, lr, batch, cosine in NET_CASES:
        res = network_train(NetworkSpec(layers, loss), ds, epochs, AdamHParams(lr=lr), seed=seed,
                            batch_size=batch, lut_size=lut_size, cosine_decay=cosine)
        probe = ds.x[:PROBE_ROWS]
        out = dict(x=ds.x.astype(np.float32), y=ds.y.astype(np.float32), epoch_losses=np.array(res.trace.epoch_losses),
                   probe_y=res.network.forward(probe))
        for i, layer in enumerate(res.network.layers):
            jod = reorder_to_jod(layer.coeff).as3d().reshape(-1)
            out[f"coeff_jod_sub_{i}"] = jod[::SUBSAMPLE_STRIDE].copy()
            out[f"coeff_jod_shape_{i}"] = np.array(reorder_to_jod(layer.coeff).as3d().shape)
            if layer.bias is not None:
                out[f"bias_{i}"] = layer.bias.copy()
        np.savez_compressed(HERE / f"train_{name}.npz", **out)
        print(name, res.trace.epoch_losses)


def main():
    for name, ds, layers, loss, epochs, lut_size, seed, lr, batch, cosine in CASES:
        res = network_train(NetworkSpec(layers, loss), ds, epochs, AdamHParams(lr=lr), seed=seed,
                            batch_size=batch, lut_size=lut_size, cosine_decay=cosine)
        out = dict(x=ds.x, y=ds.y, epoch_losses=np.array(res.trace.epoch_losses))
        for i, layer in enumerate(res.network.layers):
            out[f"coeff_jod_{i}"] = reorder_to_jod(layer.coeff).as3d().copy()
            if layer.bias is not None:
                out[f"bias_{i}"] = layer.bias.copy()
        np.savez_compressed(HERE / f"train_{name}.npz", **out)
        print(name, res.trace.epoch_losses)


if __name__ == "__main__":
    import sys

    if "--nets" in sys.argv:
        main_nets()
    else:
        main()
