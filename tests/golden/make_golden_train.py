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
    main()
