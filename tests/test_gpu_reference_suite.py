"""The reference's own tests (pkg/tests/test_pages.py, test_cache.py) run
against this package on the GPU, `kittykv` aliased to it
(tools/run_reference_suite.py; out-of-scope cases xfail with their reason).
The test files are copied next to the installed reference by
tools/install_reference.sh (git-ignored, shipped to the GPU box with the repo
snapshot); without them the test is skipped."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import kitty_oracle as ko

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_suite_against_the_package(cuda):
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref_tests")):
        pytest.skip("baseline/_ref_tests missing (tools/install_reference.sh)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "run_reference_suite.py")],
                       capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " failed" not in tail.splitlines()[-1], tail


@pytest.mark.parametrize("axis", ["per_channel", "per_token"])
@pytest.mark.parametrize("shape", [(8, 8), (13, 5), (128, 128), (1, 7)])
def test_fake_quantize_matrix_matches_oracle(cuda, axis, shape):
    # quant.py:145-177 on the device, bit-exact against the oracle's restatement
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    x = rng.normal(0, 1, shape).astype(np.float32)
    x[0, 0] = -0.0
    lanes = shape[1] if axis == "per_channel" else shape[0]
    bits = rng.choice([2, 4, 16], lanes)
    got = cuda.fake_quantize_matrix(x, axis, bits)
    want = ko.fake_quantize_matrix(x, axis, bits)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
