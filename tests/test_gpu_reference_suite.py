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


def _np_probs(keys, q):
    """cache.py:241-244 / :291-299 in numpy (float32 logits over sqrt(d), then
    the max-subtracted softmax of _softmax_columns)."""
    logits = (keys @ q) / np.float32(np.sqrt(keys.shape[-1]))
    e = np.exp(logits - logits.max(), dtype=np.float32)
    return e / e.sum()


def test_attention_probabilities(cuda):
    # oracle_attend(...).probs and KittyCacheState.attend(return_probs=True).probs
    rng = np.random.default_rng(17)
    keys = rng.normal(0, 1, (2, 300, 64)).astype(np.float32)
    values = rng.normal(0, 1, (2, 300, 64)).astype(np.float32)
    q = rng.normal(0, 1, (6, 64)).astype(np.float32)
    res = cuda.oracle_attend(keys, values, q)
    assert res.probs.shape == (6, 300)
    for i in range(6):
        np.testing.assert_allclose(res.probs[i], _np_probs(keys[i * 2 // 6], q[i]), rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(res.probs.sum(axis=1), 1.0, rtol=1e-5)
    cfg = cuda.KittyConfig(s=4, r=8, g=8, d=16, h_kv=2, h_q=4)
    st = cuda.KittyCacheState(cfg, max_tokens=64)
    k = rng.normal(0, 1, (2, 41, 16)).astype(np.float32)
    v = rng.normal(0, 1, (2, 41, 16)).astype(np.float32)
    st.prefill(k, v)
    qq = rng.normal(0, 1, (4, 16)).astype(np.float32)
    out = st.attend(qq, return_probs=True)
    assert out.probs.shape == (4, 41)
    for i in range(4):
        np.testing.assert_allclose(out.probs[i], _np_probs(st.flatten_keys(i // 2), qq[i]), rtol=1e-5, atol=1e-7)
    # the outputs are the probabilities applied to the flattened values
    for i in range(4):
        np.testing.assert_allclose(out.outputs[i], out.probs[i] @ st.flatten_values(i // 2), rtol=1e-4, atol=1e-5)
