"""Interchange formats (PKLT / PKCK / PKMX / checkpoints) against files the
reference wrote (tests/golden/make_golden_formats.py), and the file-based
``apply`` binding surface (cli.py:302-342) on the GPU."""
import json
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import GOLDEN, ROOT
from oracle import chebykan_oracle as orc
from paper_2511_14852_b200 import formats
from paper_2511_14852_b200.tensor import Layout

F = GOLDEN / "formats"


def test_pkck_roundtrip_is_byte_identical(tmp_path):
    for name in ("layer_jod.pkck", "layer_doj.pkck"):
        c = formats.load_coeff(F / name)
        assert c.layout is (Layout.JOD if "jod" in name else Layout.DOJ)
        assert (c.d_in, c.d_out, c.degree) == (12, 7, 4) and c.data.dtype == torch.float64
        formats.save_coeff(c, tmp_path / name)
        assert (tmp_path / name).read_bytes() == (F / name).read_bytes()
    jod, doj = formats.load_coeff(F / "layer_jod.pkck"), formats.load_coeff(F / "layer_doj.pkck")
    assert torch.equal(jod.as3d().permute(2, 1, 0), doj.as3d())


def test_pkmx_roundtrip_and_errors(tmp_path):
    x = formats.load_matrix(F / "x.pkmx")
    assert x.shape == (9, 12) and x.dtype == np.float64
    formats.save_matrix(x, tmp_path / "x.pkmx")
    assert (tmp_path / "x.pkmx").read_bytes() == (F / "x.pkmx").read_bytes()
    with pytest.raises(ValueError, match="matrix files hold 2-D data"):
        formats.save_matrix(np.zeros(3), tmp_path / "bad.pkmx")
    (tmp_path / "trunc.pkmx").write_bytes((F / "x.pkmx").read_bytes()[:-4])
    with pytest.raises(ValueError, match="expected 448 bytes, found 444"):
        formats.load_matrix(tmp_path / "trunc.pkmx")
    with pytest.raises(ValueError, match="not a PKMX matrix file"):
        formats.load_matrix(F / "layer_jod.pkck")


def test_pklt_reader_matches_reference_table():
    kind, degree, n, values, slopes = formats.read_lut_arrays(F / "hermite_d5_n257.pklt")
    assert kind.value == "hermite" and degree == 5 and n == 257
    want_v, want_s, _ = orc.build_table(5, 257, "hermite")
    assert np.array_equal(values, want_v.astype(np.float32).astype(np.float64))
    assert np.array_equal(slopes, want_s)


def test_pkck_errors(tmp_path):
    raw = bytearray((F / "layer_jod.pkck").read_bytes())
    raw[8] = 7  # layout tag
    (tmp_path / "bad.pkck").write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="unknown layout tag 7"):
        formats.load_coeff(tmp_path / "bad.pkck")


@pytest.mark.gpu
def test_pklt_write_matches_reference_bytes(tmp_path):
    import paper_2511_14852_b200 as ck

    t = ck.lut_build(ck.BasisKind.CHEBYSHEV, 4, 65)
    ck.save_lut(t, tmp_path / "t.pklt")
    assert (tmp_path / "t.pklt").read_bytes() == (F / "cheb_d4_n65.pklt").read_bytes()
    loaded = ck.load_lut(F / "hermite_d5_n257.pklt")
    assert loaded.kind is ck.BasisKind.HERMITE and loaded.n_features == 6
    ck.save_lut(loaded, tmp_path / "h.pklt")
    assert (tmp_path / "h.pklt").read_bytes() == (F / "hermite_d5_n257.pklt").read_bytes()


@pytest.mark.gpu
def test_checkpoint_load_and_resave_byte_identical(tmp_path):
    import paper_2511_14852_b200 as ck

    net = ck.load_checkpoint(F / "ckpt", lut_size=1024)
    assert [l.spec.kind for l in net.layers] == [ck.BasisKind.CHEBYSHEV, ck.BasisKind.LEGENDRE]
    ck.save_checkpoint(net, tmp_path / "ck")
    want = json.loads((F / "ckpt" / "manifest.json").read_text())
    got = json.loads((tmp_path / "ck" / "manifest.json").read_text())
    for lw, lg in zip(want["layers"], got["layers"]):
        bw, bg = lw.pop("bias"), lg.pop("bias")
        assert lw == lg
        np.testing.assert_allclose(bg, bw, rtol=1e-6, atol=1e-8)  # float32 device copy
    for f in ("layer_0.pkck", "layer_1.pkck"):
        assert (tmp_path / "ck" / f).read_bytes() == (F / "ckpt" / f).read_bytes()
    y = net.forward(np.linspace(-2, 2, 16).reshape(16, 1))
    assert tuple(y.shape) == (16, 1) and torch.isfinite(y).all()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["lut", "exact"])
def test_apply_cli_matches_reference_outputs(tmp_path, mode):
    cmd = [sys.executable, "-m", "paper_2511_14852_b200", "apply", "--coeff", str(F / "layer_jod.pkck"),
           "--input", str(F / "x.pkmx"), "--output", str(tmp_path / "y.pkmx"), "--bias-json", str(F / "bias.json"),
           "--mode", mode, "--lut-size", "4096", "--dy", str(F / "dy.pkmx"),
           "--coeff-grad", str(tmp_path / "cg.pkck"), "--x-grad", str(tmp_path / "xg.pkmx")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    for ours, ref in (("y.pkmx", f"y_{mode}.pkmx"), ("xg.pkmx", f"xg_{mode}.pkmx")):
        got, want = formats.load_matrix(tmp_path / ours), formats.load_matrix(F / ref)
        assert orc.normwise_err(got, want) <= 1e-4
    cg, want = formats.load_coeff(tmp_path / "cg.pkck"), formats.load_coeff(F / f"cg_{mode}.pkck")
    assert cg.layout is want.layout is Layout.DOJ
    assert orc.normwise_err(cg.data.numpy(), want.data.numpy()) <= 1e-4


@pytest.mark.gpu
def test_apply_cli_usage_and_io_errors(tmp_path):
    base = [sys.executable, "-m", "paper_2511_14852_b200", "apply", "--output", str(tmp_path / "y.pkmx")]
    r = subprocess.run(base + ["--coeff", str(tmp_path / "none.pkck"), "--input", str(F / "x.pkmx")], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 4
    formats.save_matrix(np.zeros((2, 5)), tmp_path / "x5.pkmx")
    r = subprocess.run(base + ["--coeff", str(F / "layer_jod.pkck"), "--input", str(tmp_path / "x5.pkmx")],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "input width 5 != coefficient d_in 12" in r.stderr
