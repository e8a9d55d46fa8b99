"""Reference-written interchange files (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_formats.py

Writes tests/golden/formats/: a PKLT table (save_lut, lut.py:165-177), PKCK
coefficient files in both layouts (save_coeff, tensor.py:93-104), PKMX
matrices (save_matrix, cli.py:59-68), a training checkpoint directory
(save_checkpoint, model.py:463-484), and the outputs of the reference CLI's
``apply`` on those files (cli.py:302-342) for the binding-surface test.
"""
from __future__ import annotations

import pathlib
import shutil

import numpy as np

from polykan.basis import BasisKind
from polykan.cli import main as cli_main
from polykan.cli import save_matrix
from polykan.lut import lut_build, save_lut
from polykan.model import AdamHParams, LayerSpec, NetworkSpec, make_synthetic, network_train, save_checkpoint
from polykan.tensor import CoeffTensor, Layout, reorder_to_doj, save_coeff

OUT = pathlib.Path(__file__).resolve().parent / "formats"


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir()
    save_lut(lut_build(BasisKind.HERMITE, 5, 257), OUT / "hermite_d5_n257.pklt")
    save_lut(lut_build(BasisKind.CHEBYSHEV, 4, 65), OUT / "cheb_d4_n65.pklt")
    rng = np.random.default_rng(4)
    d_in, d_out, degree = 12, 7, 4
    c = CoeffTensor(d_in, d_out, degree, Layout.JOD, rng.uniform(-0.2, 0.2, d_in * d_out * (degree + 1)))
    save_coeff(c, OUT / "layer_jod.pkck")
    save_coeff(reorder_to_doj(c), OUT / "layer_doj.pkck")
    x = rng.uniform(-2, 2, (9, d_in)).astype(np.float32)
    dy = rng.standard_normal((9, d_out)).astype(np.float32)
    save_matrix(x, OUT / "x.pkmx")
    save_matrix(dy, OUT / "dy.pkmx")
    (OUT / "bias.json").write_text("[" + ", ".join(repr(float(v)) for v in rng.uniform(-0.1, 0.1, d_out)) + "]")
    for mode in ("lut", "exact"):
        code = cli_main(["apply", "--coeff", str(OUT / "layer_jod.pkck"), "--input", str(OUT / "x.pkmx"),
                         "--output", str(OUT / f"y_{mode}.pkmx"), "--bias-json", str(OUT / "bias.json"),
                         "--mode", mode, "--lut-size", "4096", "--dy", str(OUT / "dy.pkmx"),
                         "--coeff-grad", str(OUT / f"cg_{mode}.pkck"), "--x-grad", str(OUT / f"xg_{mode}.pkmx")])
        assert code == 0
    res = network_train(NetworkSpec((LayerSpec(1, 4, 3), LayerSpec(4, 1, 3, BasisKind.LEGENDRE))),
                        make_synthetic("cheb2"), 1, AdamHParams(lr=1e-2), seed=2, lut_size=1024)
    save_checkpoint(res.network, OUT / "ckpt")
    print(sorted(p.name for p in OUT.rglob("*")))


if __name__ == "__main__":
    main()
