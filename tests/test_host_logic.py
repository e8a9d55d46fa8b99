"""Host-side logic of the product package (no GPU): schedule validation,
layouts, LUT sizing, sharding -- mirroring the reference's own unit tests."""
import numpy as np
import pytest
import torch

from oracle import chebykan_oracle as orc
from paper_2511_14852_b200 import (
    DEFAULT_LUT_SIZE,
    ChebyKANLayer,
    CoeffTensor,
    Layout,
    TileSchedule,
    doj_index,
    interp_error_bound,
    jod_index,
    lut_size_for_budget,
    reorder_to_doj,
    reorder_to_jod,
    shard_bounds,
)


def test_default_lut_size_is_reference_default():
    assert DEFAULT_LUT_SIZE == orc.REFERENCE_DEFAULT_LUT_SIZE == 32768


def test_schedule_invariants():  # test_kernels.py:417-425
    with pytest.raises(ValueError, match="tile_out == lane_y"):
        TileSchedule(tile_in=8, tile_out=8, lane_x=4, lane_y=16, g_x=1, g_y=1, d_in=8, d_out=8)
    with pytest.raises(ValueError, match="g_x"):
        TileSchedule(tile_in=8, tile_out=8, lane_x=4, lane_y=8, g_x=3, g_y=1, d_in=8, d_out=8)
    s = TileSchedule.for_dims(100, 70, tile_in=16, tile_out=32)
    assert s.g_x == 7 and s.g_y == 3
    with pytest.raises(ValueError):
        TileSchedule.for_dims(0, 4)


def test_layout_index_maps_and_reorder_roundtrip():  # tensor.py:67-90
    d_in, d_out, deg = 5, 3, 4
    k = deg + 1
    jod = torch.arange(d_in * d_out * k, dtype=torch.float32)
    c = CoeffTensor(d_in, d_out, deg, Layout.JOD, jod)
    doj = reorder_to_doj(c)
    flat = doj.data.reshape(-1)
    for j in range(d_in):
        for o in range(d_out):
            for kk in range(k):
                assert flat[doj_index(d_in, d_out, kk, o, j)] == jod[jod_index(d_out, deg, j, o, kk)]
    back = reorder_to_jod(doj)
    assert torch.equal(back.data.reshape(-1), jod)
    with pytest.raises(ValueError, match="expects JOD"):
        reorder_to_doj(doj)
    with pytest.raises(ValueError, match="expected"):
        CoeffTensor(2, 2, 1, Layout.JOD, torch.zeros(7))


def test_interp_bound_matches_oracle():
    for d, n in ((8, 1024), (3, 512), (15, 16384), (24, 32768)):
        assert np.array_equal(interp_error_bound(d, n), orc.interp_error_bound(d, n))


def test_lut_size_for_budget():
    for d in (3, 5, 8, 15):
        n = lut_size_for_budget(d, 1e-4)
        assert interp_error_bound(d, n).max() <= 1e-4
        assert n == 2 or interp_error_bound(d, n // 2).max() > 1e-4


def test_shard_bounds_partition():
    for gb, w in ((262144, 8), (1000, 3), (5, 8)):
        covered = []
        for r in range(w):
            a, b = shard_bounds(gb, r, w)
            covered.extend(range(a, b))
        assert covered == list(range(gb))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_layer_init_matches_reference_init_params():  # model.py:72-83
    layer = ChebyKANLayer(6, 4, 3, seed=123)
    rng = np.random.default_rng(123)
    s = 1.0 / np.sqrt(6 * 4)
    want = rng.uniform(-s, s, size=6 * 4 * 4).reshape(6, 4, 4).astype(np.float32)
    assert np.array_equal(layer.cheby_coeffs.detach().numpy(), want)
    assert torch.count_nonzero(layer.bias) == 0
    assert tuple(layer.coeff_doj.shape) == (4, 4, 6)
    with pytest.raises(ValueError):
        ChebyKANLayer(0, 4, 3)


def test_layer_refuses_cpu_tensors():
    layer = ChebyKANLayer(4, 2, 2)
    with pytest.raises(ValueError, match="CUDA"):
        layer(torch.zeros(3, 4))


def test_model_specs_validate_like_reference():
    import paper_2511_14852_b200 as ck

    with pytest.raises(ValueError, match="layer dimensions must be >= 1"):
        ck.LayerSpec(0, 3, 2)
    with pytest.raises(ValueError, match="degree must be >= 0"):
        ck.LayerSpec(2, 3, -1)
    with pytest.raises(ValueError, match="layer dims do not chain: 3 -> 4"):
        ck.NetworkSpec((ck.LayerSpec(2, 3, 1), ck.LayerSpec(4, 1, 1)))
    with pytest.raises(ValueError, match="a network needs at least one layer"):
        ck.NetworkSpec(())
    assert ck.LayerSpec(2, 3, 4, ck.BasisKind.FOURIER).n_feat == 9


def test_synthetic_datasets_match_reference_fixtures():
    import numpy as np

    import paper_2511_14852_b200 as ck
    from conftest import GOLDEN

    g = np.load(GOLDEN / "train_cheb2.npz")
    ds = ck.make_synthetic("cheb2")
    assert np.array_equal(ds.x, g["x"]) and np.array_equal(ds.y, g["y"])
    with pytest.raises(ck.DatasetError, match="unknown synthetic dataset 'nope'; known: cheb2, sincos"):
        ck.make_synthetic("nope")


def test_roofline_formulas_match_reference():
    # test_acceptance.py:279-298 (closed forms of perf.py:77-90) and the CLI
    # lambda case of test_cli.py:100-113
    import numpy as np

    import paper_2511_14852_b200 as ck

    r = ck.roofline(ck.LayerConfig(128, 40, 256, 8, 4))
    assert r.flops == 23_674_880 and r.bytes == 888_832
    assert abs(r.intensity - 23_674_880 / 888_832) < 1e-9
    rng = np.random.default_rng(1006)
    for _ in range(200):
        b, din, dout = (int(rng.integers(1, v)) for v in (512, 2048, 2048))
        d, lam = int(rng.integers(0, 33)), int(rng.choice([4, 8]))
        rep = ck.roofline(ck.LayerConfig(b, din, dout, d, lam))
        assert rep.flops == 2 * b * din * (d + (d + 1) * dout)
        assert rep.bytes == lam * (b * din + b * dout + 2 * b * din * (d + 1) + din * dout * (d + 1))
    assert ck.roofline(ck.LayerConfig(2, 3, 4, 1, 8)).bytes == 2 * 4 * (2 * 3 + 2 * 4 + 2 * 2 * 3 * 2 + 3 * 4 * 2)
    assert [c.degree for c in ck.paper_configs()] == [8, 15, 24]
    with pytest.raises(ValueError, match="elem_bytes"):
        ck.LayerConfig(1, 1, 1, 1, 2)


def test_reference_public_names_are_exported():
    # every name polykan/__init__.py exports (its public surface, __init__.py:8-83)
    import paper_2511_14852_b200 as ck

    names = """BasisKind RecurrenceCoeffs eval_basis eval_basis_derivative eval_basis_trig feature_count
    AtomicCounts BasisPath EXACT_MODE KernelCounters KernelMode LUT_MODE NonFiniteInputError PartialBuffer
    TileSchedule backward_fused combine count_atomics forward_partial fused_forward reference_forward
    DEFAULT_LUT_SIZE LutTable load_lut lut_build lut_interp lut_interp_with_slope lut_max_error_bound save_lut
    AdamHParams AdamState Dataset Layer LayerSpec Loss Network NetworkSpec init_params layer_forward
    load_checkpoint make_synthetic network_train save_checkpoint
    BenchResult LayerConfig Regime RooflineReport paper_configs roofline run_bench
    CoeffTensor Layout doj_index jod_index load_coeff reorder_to_doj reorder_to_jod
    save_coeff""".split()
    missing = [n for n in names if not hasattr(ck, n)]
    assert not missing, missing
