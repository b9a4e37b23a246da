"""The C oracle against the golden fixtures of tests/golden/make_golden.py (an
independent pure-Python restatement: 40-digit GLL operators, exact-fma sweeps,
sort-based selection in Python integers, stream layout of include/isf_lossy.h)."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v2.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.mark.parametrize("lx", range(2, 17))
def test_operators_match_golden(oracle, golden, lx):
    F, B = oracle.matrices(lx)
    x, w = oracle.gll(lx)
    assert np.array_equal(F, golden[f"F{lx}"])
    assert np.array_equal(B, golden[f"B{lx}"])
    assert np.array_equal(x, golden[f"x{lx}"])
    assert np.array_equal(w, golden[f"w{lx}"])


def test_streams_match_golden(oracle, golden):
    for name in golden["cases"]:
        lx, eps = golden[f"{name}__meta"]
        lx = int(lx)
        field = golden[f"{name}__field"]
        co = oracle.forward_field(field, lx, 1)
        assert np.array_equal(co, golden[f"{name}__coeffs"]), name
        rc, s, st = oracle.compress(field, lx, 1, float(eps))
        assert rc == 0
        assert np.array_equal(s, golden[f"{name}__stream"]), name


def test_golden_generator_is_reproducible(tmp_path):
    # the committed fixture is what the committed script produces
    import importlib.util
    import shutil
    src = os.path.join(os.path.dirname(__file__), "golden", "make_golden.py")
    dst = tmp_path / "make_golden.py"
    shutil.copy(src, dst)
    spec = importlib.util.spec_from_file_location("mg", dst)
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    mg.main()
    a = np.load(GOLDEN)
    b = np.load(tmp_path / "golden_v2.npz")
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
