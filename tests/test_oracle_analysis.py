"""The oracle's restatement of the analysis row (analysis.py:63-142) against
golden vectors made by the reference itself (tests/golden/make_golden_analysis.py)."""

import os

import numpy as np
import pytest

from oracle import kitty_oracle as ko

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_analysis.npz")


@pytest.fixture(scope="module")
def ga():
    return dict(np.load(GOLDEN))


def test_sensitivity_oracle_matches_reference(ga):
    for i in range(int(ga["num_sens"][0])):
        if ga[f"sens{i}_q"].shape[-1] > 64:
            continue  # the 128-channel case is checked on the device only (seconds in numpy)
        mse = ko.channel_sensitivity(ga[f"sens{i}_q"], ga[f"sens{i}_k"], int(ga[f"sens{i}_bits"][0]))
        np.testing.assert_allclose(mse, ga[f"sens{i}_mse"], rtol=1e-9, atol=1e-18)
        assert np.array_equal(np.argsort(-mse, axis=1, kind="stable"), ga[f"sens{i}_ranking"]), i


def test_constant_channel_is_exactly_zero(ga):
    assert np.all(ga["sens1_mse"][:, 5] == 0.0)
    assert np.all(ko.channel_sensitivity(ga["sens1_q"], ga["sens1_k"])[:, 5] == 0.0)


def test_attention_mse_oracle_matches_reference(ga):
    for i in range(int(ga["num_sweep"][0])):
        k, q = ga[f"sweep{i}_k"], ga[f"sweep{i}_q"]
        np.testing.assert_allclose(ko.attention_mse(k, q, ga[f"sweep{i}_sel"]), ga[f"sweep{i}_mse_sel"][0], rtol=1e-12)
        np.testing.assert_allclose(ko.attention_mse(k, q, []), ga[f"sweep{i}_mse_none"][0], rtol=1e-12)
