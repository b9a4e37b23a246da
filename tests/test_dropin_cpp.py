"""C++ drop-in: include/isf/tasks/lossy.hpp compiled against the reference's own
core headers and sources (/root/reference/proj) and linked with libisf_lossy.so
(`make -C oracle dropin`).  The binary is built here (CPU) and run on the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin")


def test_dropin_builds_against_reference_headers():
    if not os.path.isdir("/root/reference/proj"):
        pytest.skip("reference sources not present (GPU box)")
    from paper_2407_20731_b200 import build as B
    B.build()
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("drop-in binary not built (build() on the CPU container builds it)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok=1" in r.stdout
