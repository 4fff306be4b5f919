"""The golden pipeline reproduces: tests/golden/make_golden.py run against the unmodified
reference regenerates every committed fixture bit for bit (NaN-aware).  Needs the reference
(dev container: /root/reference); skipped where it is absent (the GPU box)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from cases import GOLDEN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src/strom"), reason="reference not present")
def test_make_golden_regenerates_every_fixture(tmp_path):
    env = dict(os.environ, GOLDEN_OUT=str(tmp_path), OPENBLAS_NUM_THREADS="1")
    r = subprocess.run([sys.executable, os.path.join(GOLDEN, "make_golden.py")], env=env, capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    committed = sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz"))
    assert sorted(f for f in os.listdir(tmp_path) if f.endswith(".npz")) == committed
    for f in committed:
        with np.load(os.path.join(GOLDEN, f)) as a, np.load(os.path.join(tmp_path, f)) as b:
            assert sorted(a.files) == sorted(b.files), f
            for k in a.files:
                x, y = a[k], b[k]
                assert x.shape == y.shape and np.array_equal(x, y, equal_nan=x.dtype.kind == "f"), (f, k)
