"""SPEC.md:240-248 lossless stage (include/isf/tasks/lossless.hpp): RLE of 1 MiB of
zeros has cr >= 0.99, every codec round-trips random bytes exactly, Eq. 1 gives 0 for
equal sizes, an unknown codec id raises UnknownCodec (tests/cpp/lossless_main.cpp,
`make -C oracle lossless`, CPU only)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "lossless")


def test_lossless_codecs():
    if os.path.isdir("/root/reference/proj"):
        from paper_2407_20731_b200 import build as B
        B.build()
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "lossless"], capture_output=True,
                           text=True)
        assert r.returncode == 0, r.stderr
    if not os.path.exists(BIN):
        pytest.skip("lossless binary not built (needs the reference sources)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert json.loads(r.stdout.strip().splitlines()[-1])["ok"]
