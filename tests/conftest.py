import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
if os.path.join(ROOT, "oracle") not in sys.path:
    sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_names():
    return sorted(
        os.path.basename(p)[:-4]
        for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
        if not os.path.basename(p).startswith(("decisions", "cfg"))
    )


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def assert_same_topk(ids, scores, want_ids, want_scores, rtol=1e-9, atol=1e-9, ctx=""):
    """Reference tests/conftest.py:41-47 semantics: identical ids in identical
    order, scores equal up to kernel rounding."""
    __tracebackhide__ = True
    ids = np.asarray(ids)
    want_ids = np.asarray(want_ids)
    assert ids.shape == want_ids.shape, f"{ctx}: shape {ids.shape} != {want_ids.shape}"
    bad = np.flatnonzero((ids != want_ids).any(axis=-1)) if ids.ndim == 2 else (
        [0] if not np.array_equal(ids, want_ids) else [])
    assert len(bad) == 0, f"{ctx}: {len(bad)} rows differ, first row {bad[0]}: {ids[bad[0]]} vs {want_ids[bad[0]]}"
    np.testing.assert_allclose(scores, want_scores, rtol=rtol, atol=atol, err_msg=ctx)


def canonical_ids(items, ids):
    """Map each item id to the lowest id with a bit-identical vector
    (reference tests/conftest.py:57-67)."""
    rep = {}
    first = np.empty(items.shape[0], dtype=np.int64)
    for i in range(items.shape[0]):
        first[i] = rep.setdefault(items[i].tobytes(), i)
    return first[np.asarray(ids)]


def near_tie_rows(scores_sorted_full, k, rel=1e-5):
    """Rows whose K-th and (K+1)-th exact scores lie within ``rel`` (the judge's
    tie clause); ids may legitimately differ at such boundaries."""
    s = scores_sorted_full
    if s.shape[1] <= k:
        return np.zeros(s.shape[0], dtype=bool)
    a, b = s[:, k - 1], s[:, k]
    return np.abs(a - b) <= rel * np.maximum(np.abs(a), 1e-30)


@pytest.fixture(scope="session")
def oracle():
    import simdex_oracle
    return simdex_oracle


def assert_lists_equal_up_to_ties(ids, bounds, want_ids, want_bounds, rel=1e-12, ctx=""):
    """Index lists equal, except that items whose ceilings agree to ``rel``
    (mathematical ties that float64 rounding orders arbitrarily) may appear in
    any order within their run."""
    __tracebackhide__ = True
    np.testing.assert_allclose(bounds, want_bounds, rtol=rel, atol=rel, err_msg=ctx)
    for c in range(want_ids.shape[0]):
        wb = want_bounds[c]
        brk = np.flatnonzero(np.abs(np.diff(wb)) > rel * np.maximum(np.abs(wb[1:]), 1.0)) + 1
        for seg in np.split(np.arange(wb.shape[0]), brk):
            assert set(ids[c][seg].tolist()) == set(want_ids[c][seg].tolist()), f"{ctx} cluster {c} run {seg[:3]}"
