"""CPU tests: the C-ABI library loads and exports every declared symbol,
rejects bad arguments without touching a device, and the host-side logic of
the package (decision rule, config, model I/O, validation) matches the
reference's contracts."""

import ctypes
import math
import os

import numpy as np
import pytest

from conftest import load_golden

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib
from paper_1706_01449_b200 import optimizer as opt


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"
    assert lib.simdex_abi_version() == 1


def test_abi_rejects_bad_arguments_without_a_device():
    lib = _lib.load()
    rc = lib.simdex_topk_exact(None, 10, None, 10, 4, None, 10, 3, None, None, None)
    assert rc == -1
    assert b"null pointer" in lib.simdex_last_error()
    buf = (ctypes.c_double * 16)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    rc = lib.simdex_walk(p, p, p, 4, 0, p, p, p, p, 1, 3, 0, None, None, None, 0, p, p, p, None)
    assert rc == -1 and b"bad sizes" in lib.simdex_last_error()
    rc = lib.simdex_walk(p, p, p, 4, 8, p, p, p, p, 1, 3, 5, None, None, None, 0, p, p, p, None)
    assert rc == -1 and b"warm start" in lib.simdex_last_error()
    rc = lib.simdex_merge_topk(p, p, 0, 1, 1, 1, p, p, None)
    assert rc == -1


def test_product_path_refuses_without_cuda(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    model = sx.ModelPair(sx.FactorMatrix(np.ones((3, 2))), sx.FactorMatrix(np.ones((4, 2))))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sx.topk_matmul(model, 2)


def test_validation_before_device():
    model = sx.ModelPair(sx.FactorMatrix(np.ones((3, 2))), sx.FactorMatrix(np.ones((4, 2))))
    for fn in (sx.topk_matmul, sx.topk_naive):
        with pytest.raises(ValueError):
            fn(model, 0)
    with pytest.raises(ValueError):
        sx.kmeans(model.users, 4)
    with pytest.raises(ValueError):
        sx.kmeans(model.users, 0)
    with pytest.raises(ValueError):
        sx.kmeans(model.users, 2, max_iters=0)
    with pytest.raises(ValueError):
        sx.run_pipeline(model, k=1, force="both")
    with pytest.raises(ValueError):
        sx.BlockSpec(0, 4)
    with pytest.raises(sx.DimensionMismatchError):
        sx.ModelPair(sx.FactorMatrix(np.ones((3, 2))), sx.FactorMatrix(np.ones((4, 3))))
    with pytest.raises(sx.NonFiniteValueError):
        sx.FactorMatrix(np.array([[1.0, np.nan]]))
    with pytest.raises(sx.FormatError):
        sx.FactorMatrix(np.ones(3))
    with pytest.raises(ValueError):
        sx.item_bound(-1.0, 0.5, 0.5)
    with pytest.raises(ValueError):
        sx.item_bound(1.0, -0.1, 0.0)


def test_decision_rule_matches_reference_table():
    g = load_golden("decisions")
    n = 1 << 20
    for row, picks in zip(g["fractions"], g["picks"]):
        for f, k, want in zip(row, (1, 5, 10, 50), picks):
            assert sx.decide(f * n, n, 0, k, 0.05) == want
    np.testing.assert_allclose([sx.hardware_factor(k, 0.05) for k in (1, 2, 5, 10, 50, 500)], g["hw_factor"])
    assert sx.decide(0.05 * 1024, 1024, 0, 1, 0.05) == sx.INDEX          # boundary inclusive
    assert sx.decide(1.0, 100, 100, 1, 0.9) == sx.MATMUL
    assert sx.pruning_fraction(10.0, 1000, 100) == 0.0
    assert sx.pruning_fraction(10_000.0, 1000, 100) == 1.0
    with pytest.raises(ValueError):
        sx.hardware_factor(0, 0.05)
    with pytest.raises(ValueError):
        sx.hardware_factor(5, 0.0)
    assert math.floor(sx.hardware_factor(10) * 100) / 100 == 0.16


def test_config_round_trip(tmp_path, monkeypatch):
    path = tmp_path / "cfg"
    opt.save_config(path, {"h0": 0.031, "clusters": 8, "note": "local"})
    assert opt.load_config(path) == {"h0": 0.031, "clusters": 8, "note": "local"}
    opt.save_config(path, {"h0": 0.2})
    monkeypatch.setenv(opt.CONFIG_ENV, str(path))
    assert opt.resolve_h0(0.4) == 0.4
    assert opt.resolve_h0(None) == 0.2
    monkeypatch.delenv(opt.CONFIG_ENV)
    assert opt.resolve_h0(None) == opt.DEFAULT_H0


SPECS = [  # the golden cases' SyntheticSpecs (oracle/make_golden.py small_cases)
    ("syn0", (50, 140, 6, 8, 0.3, (0.3, 3.0), 3)),
    ("syn1", (200, 500, 8, 6, 0.5, (0.5, 2.5), 42)),
    ("syn6", (25, 33, 1, 2, 0.0, (0.5, 2.0), 6)),
]


@pytest.mark.parametrize("name,spec", SPECS)
def test_generate_synthetic_matches_reference(name, spec):
    nu, ni, f, a, s, nr, seed = spec
    m = sx.generate_synthetic(sx.SyntheticSpec(nu, ni, f, archetype_count=min(a, nu), angular_spread=s,
                                               norm_low=nr[0], norm_high=nr[1], seed=seed))
    g = load_golden(name)
    np.testing.assert_array_equal(m.users.values, g["users"])
    np.testing.assert_array_equal(m.items.values, g["items"])


def test_matrix_files_round_trip(tmp_path):
    m = sx.generate_synthetic(sx.SyntheticSpec(20, 30, 4, seed=1))
    sx.save_model(m, tmp_path / "u.mf", tmp_path / "i.mf")
    back = sx.load_model(tmp_path / "u.mf", tmp_path / "i.mf")
    assert np.array_equal(back.users.values, m.users.values) and np.array_equal(back.items.values, m.items.values)
    (tmp_path / "c.csv").write_text("1,2\n3,4\n")
    assert sx.load_matrix(tmp_path / "c.csv").values.tolist() == [[1.0, 2.0], [3.0, 4.0]]
    (tmp_path / "bad.csv").write_text("1,2\n3\n")
    with pytest.raises(sx.DimensionMismatchError):
        sx.load_matrix(tmp_path / "bad.csv")
    (tmp_path / "bad.bin").write_bytes(b"MFMAT001" + b"\0" * 10)
    with pytest.raises(sx.FormatError):
        sx.load_matrix(tmp_path / "bad.bin")


def test_results_sequence_semantics():
    ids = np.array([[3, 1], [0, 2]], dtype=np.int32)
    sc = np.array([[2.0, 1.0], [5.0, 4.0]])
    cached = sx.TopKResult(7, np.array([1, 2]), np.array([9.0, 8.0]), 3)
    res = sx.TopKResults([5, 7], ids, sc, np.array([4, 4]), {1: cached})
    assert len(res) == 2 and res[1] is cached and res[-1] is cached
    r0 = res[0]
    assert r0.user_id == 5 and r0.item_ids.dtype == np.int64 and r0.scores.dtype == np.float64
    assert r0.entries == [(3, 2.0), (1, 1.0)]
    assert [r.user_id for r in res] == [5, 7]
    with pytest.raises(IndexError):
        res[2]
