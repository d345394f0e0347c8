import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_02382_b200 import _native

    _native.load()  # fail loudly if the native library is missing
    return torch.device("cuda:0")


def nerr(a, b):
    """Normalized max error max|a-b| / max|b|."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def assert_close_ref(got, want, tol, name=""):
    """The reference's acceptance form |a-b| <= tol + tol*|b| (test_acceptance.py:58-64),
    applied after normalising by max|b| so tiny absolute noise (e.g. the
    mathematically-zero K bias gradient) passes."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    bad = np.abs(got - want) > tol * scale + tol * np.abs(want)
    assert not bad.any(), f"{name}: {bad.sum()} elements out of tolerance {tol}, nerr={nerr(got, want):.3e}"


def free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def ns_inputs(seq, embed=1024, seed=0):
    """Inputs of the north-star-shape fixtures (tests/golden/ns_inputs.py)."""
    sys.path.insert(0, str(GOLDEN_DIR))
    from ns_inputs import ns_inputs as gen

    return gen(seq, embed, seed=seed)


def check_ns_golden(z, y, dx, grads, tol, name=""):
    """Compare a full result (y, dx (B, l, E); grads {reference name: array}) with an
    NS fixture (tests/golden/make_golden.py ns_case): the stored row subsets in the
    reference's |a-b| <= tol*max|b| + tol*|b| form, and the row-sum checksums (which
    cover every element) normalised by the sum of absolute values they fold."""
    sys.path.insert(0, str(GOLDEN_DIR))
    from ns_inputs import ATTN_NAMES, ROW_STRIDE, WROW_STRIDE

    y, dx = np.asarray(y, np.float64), np.asarray(dx, np.float64)
    assert_close_ref(y[:, ::ROW_STRIDE], z["y_rows"], tol, f"{name} y rows")
    assert_close_ref(dx[:, ::ROW_STRIDE], z["dx_rows"], tol, f"{name} dx rows")
    for what, full, key in (("y", y, "y_rowsum"), ("dx", dx, "dx_rowsum")):
        scale = np.abs(full).sum(-1).max()
        err = np.abs(full.sum(-1) - z[key]).max() / scale
        assert err < tol, f"{name} {what} row sums: {err:.3e}"
    for nm in ATTN_NAMES:
        g = np.asarray(grads[nm], np.float64)
        if g.ndim == 1:
            if nm == "bk":  # mathematically zero (softmax shift invariance): absolute check
                assert np.abs(g).max() <= tol * np.abs(z["g_wk_rows"]).max(), f"{name} bk"
                continue
            assert_close_ref(g, z["g_" + nm], tol, f"{name} {nm}")
            continue
        assert_close_ref(g[::WROW_STRIDE], z["g_" + nm + "_rows"], tol, f"{name} {nm} rows")
        for ax, key in ((1, "_rowsum"), (0, "_colsum")):
            scale = np.abs(g).sum(ax).max()
            err = np.abs(g.sum(ax) - z["g_" + nm + key]).max() / scale
            assert err < tol, f"{name} {nm}{key}: {err:.3e}"
