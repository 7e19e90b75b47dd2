"""GPU parity of the analysis row (analysis.py:63-236):
channel_sensitivity / attention_mse / boost_sweep / boost_sweep_experiment
run through kitty_channel_sensitivity / kitty_attention_mse, against golden
vectors made by the reference (tests/golden/make_golden_analysis.py) and the
reference's own known-answer tests (test_analysis.py:32-141).

Bar: fp64 values within rtol 1e-9 of the reference (the reference's own
tolerance for the rank-1 update vs direct recomputation, test_analysis.py:61);
rankings identical; the exact identities (constant channel, bits 16,
full-boost / zero-boost sweeps) exactly."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_analysis.npz")


@pytest.fixture(scope="module")
def ga():
    return dict(np.load(GOLDEN))


def test_sensitivity_matches_reference_golden(cuda, ga):
    for i in range(int(ga["num_sens"][0])):
        rep = cuda.channel_sensitivity(ga[f"sens{i}_q"], ga[f"sens{i}_k"], bits=int(ga[f"sens{i}_bits"][0]))
        np.testing.assert_allclose(rep.mse, ga[f"sens{i}_mse"], rtol=1e-9, atol=1e-18, err_msg=str(i))
        assert np.array_equal(rep.ranking, ga[f"sens{i}_ranking"]), i
        assert rep.mse.shape == ga[f"sens{i}_mse"].shape


def test_constant_channel_zero_and_passthrough(cuda):
    # test_analysis.py:32-47
    rng = np.random.default_rng(0)
    keys = rng.normal(0, 1, (40, 8)).astype(np.float32)
    keys[:, 5] = 1.5
    queries = rng.normal(0, 1, (16, 8)).astype(np.float32)
    rep = cuda.channel_sensitivity(queries, keys)
    assert rep.mse[0, 5] == 0.0 and np.all(rep.mse >= 0)
    assert np.all(cuda.channel_sensitivity(queries, keys, bits=16).mse == 0.0)


def test_outlier_channels_rank_top(cuda):
    # test_analysis.py:66-74
    keys = cuda.generate_synthetic(cuda.SyntheticSpec(tokens=1024, channels=32, outlier_channels=(3, 17),
                                                      outlier_gain=8.0, seed=3))
    queries = np.random.default_rng(4).normal(0, 1, (2, 64, 32)).astype(np.float32)
    assert set(cuda.channel_sensitivity(queries, keys).top_channels(2).tolist()) == {3, 17}


def test_permutation_invariance_and_gqa_shapes(cuda):
    # test_analysis.py:77-101
    rng = np.random.default_rng(5)
    keys = rng.normal(0, 1, (30, 8)).astype(np.float32)
    queries = rng.normal(0, 1, (15, 8)).astype(np.float32)
    perm = np.array([7, 1, 2, 0, 6, 5, 4, 3])
    a = cuda.channel_sensitivity(queries, keys).mse[0, 2]
    b = cuda.channel_sensitivity(queries[:, perm], keys[:, perm]).mse[0, 2]
    np.testing.assert_allclose(b, a, rtol=1e-6, atol=1e-18)
    rep = cuda.channel_sensitivity(rng.normal(0, 1, (4, 10, 8)).astype(np.float32),
                                   rng.normal(0, 1, (2, 20, 8)).astype(np.float32))
    assert rep.mse.shape == (4, 8) and rep.ranking.shape == (4, 8)
    with pytest.raises(cuda.KittyError):
        cuda.channel_sensitivity(rng.normal(0, 1, (3, 10, 8)).astype(np.float32),
                                 rng.normal(0, 1, (2, 20, 8)).astype(np.float32))


def test_attention_mse_and_sweep_match_reference(cuda, ga):
    for i in range(int(ga["num_sweep"][0])):
        k, q = ga[f"sweep{i}_k"], ga[f"sweep{i}_q"]
        np.testing.assert_allclose(cuda.attention_mse(k, q, ga[f"sweep{i}_sel"]), ga[f"sweep{i}_mse_sel"][0], rtol=1e-9)
        np.testing.assert_allclose(cuda.attention_mse(k, q, []), ga[f"sweep{i}_mse_none"][0], rtol=1e-9)
        want = ga[f"sweep{i}_rows"]
        fr = sorted({float(r[0]) for r in want})
        frac = [f for f in fr if f not in (0.0, 0.0625, 0.5)]
        rows = cuda.boost_sweep(k, q, [0.0, 0.0625] + frac + [0.5], random_draws=3, seed=[7, 8, 9][i])
        got = np.array([[r.fraction, r.heuristic == "magnitude", r.mean_mse, r.max_deviation, r.runs] for r in rows])
        assert got.shape == want.shape
        np.testing.assert_array_equal(got[:, [0, 1, 4]], want[:, [0, 1, 4]])
        np.testing.assert_allclose(got[:, 2], want[:, 2], rtol=1e-9)
        np.testing.assert_allclose(got[:, 3], want[:, 3], rtol=1e-6, atol=1e-15)


def test_sweep_identities(cuda):
    # test_analysis.py:104-120
    rng = np.random.default_rng(7)
    keys = rng.normal(0, 1, (64, 16)).astype(np.float32)
    queries = rng.normal(0, 1, (16, 16)).astype(np.float32)
    by = {r.heuristic: r for r in cuda.boost_sweep(keys, queries, [1.0], random_draws=3)}
    assert by["magnitude"].mean_mse == by["random"].mean_mse and by["random"].max_deviation == 0.0
    rng = np.random.default_rng(8)
    keys = rng.normal(0, 1, (64, 16)).astype(np.float32)
    queries = rng.normal(0, 1, (16, 16)).astype(np.float32)
    uniform = cuda.attention_mse(keys, queries, [])
    assert all(r.mean_mse == uniform for r in cuda.boost_sweep(keys, queries, [0.0], random_draws=2))


def test_experiment_matches_reference_and_orders(cuda, ga):
    # test_analysis.py:131-141
    rows = cuda.boost_sweep_experiment([0.0, 0.125, 0.25], n_seeds=3, tokens=256, channels=32,
                                       outlier_channels=(3, 17), query_tokens=32)
    got = np.array([[r.fraction, r.heuristic == "magnitude", r.mean_mse, r.max_deviation, r.runs] for r in rows])
    want = ga["experiment_rows"]
    np.testing.assert_array_equal(got[:, [0, 1, 4]], want[:, [0, 1, 4]])
    np.testing.assert_allclose(got[:, 2], want[:, 2], rtol=1e-9)
    by = {(r.fraction, r.heuristic): r.mean_mse for r in rows}
    assert by[(0.125, "magnitude")] <= by[(0.125, "random")]
    assert by[(0.0, "magnitude")] >= by[(0.125, "magnitude")] >= by[(0.25, "magnitude")]


def test_sensitivity_at_decode_shape(cuda):
    # a LLaMA3-8B KV head's page-sized sensitivity scan: 4 query heads x 64
    # query tokens over 4096 keys x 128 channels; outlier channels rank top
    keys = cuda.generate_synthetic(cuda.SyntheticSpec(tokens=4096, channels=128, outlier_channels=(9, 40, 77),
                                                      outlier_gain=8.0, seed=1))
    queries = np.random.default_rng(2).normal(0, 1, (4, 64, 128)).astype(np.float32)
    rep = cuda.channel_sensitivity(queries, keys)
    assert set(rep.top_channels(3).tolist()) == {9, 40, 77}
