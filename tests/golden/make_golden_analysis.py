"""Golden vectors for the analysis row from the REFERENCE
implementation (kittykv.analysis), generated in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_analysis.py

writes ``tests/golden/golden_analysis.npz``: channel_sensitivity reports
(mse, ranking) for MHA and GQA shapes including a constant channel and
outlier channels, attention_mse of explicit selections, boost_sweep rows (both
heuristics) and a small boost_sweep_experiment.  Nothing here runs on the GPU
box; the GPU tests compare the device against these arrays.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import kittykv as kv  # noqa: E402
from kittykv import analysis as an  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_analysis.npz")

# (h_q, lq, h_kv, L, d, bits, seed)
SENS = [
    (1, 12, 1, 24, 8, 2, 2),
    (1, 16, 1, 40, 8, 2, 0),  # channel 5 constant (test_analysis.py:32-39)
    (4, 10, 2, 20, 8, 2, 6),
    (2, 64, 1, 1024, 32, 2, 3),  # outlier channels 3, 17 (test_analysis.py:66-74)
    (8, 16, 2, 300, 128, 2, 11),
    (2, 8, 2, 200, 64, 4, 12),
]
# (L, d, heads, lq, fraction, seed)
SWEEP = [(64, 16, 1, 16, 0.25, 7), (256, 32, 2, 32, 0.125, 8), (1024, 128, 1, 64, 0.125, 9)]


def main():
    out = {}
    for i, (h_q, lq, h_kv, L, d, bits, seed) in enumerate(SENS):
        rng = np.random.default_rng(seed)
        if i == 3:
            keys = kv.generate_synthetic(kv.SyntheticSpec(tokens=L, channels=d, outlier_channels=(3, 17),
                                                          outlier_gain=8.0, seed=3))[None]
        else:
            keys = rng.normal(0, 1 + i % 2, (h_kv, L, d)).astype(np.float32)
        if i == 1:
            keys[:, :, 5] = 1.5
        queries = rng.normal(0, 1, (h_q, lq, d)).astype(np.float32)
        rep = an.channel_sensitivity(queries, keys, bits=bits)
        out[f"sens{i}_q"] = queries
        out[f"sens{i}_k"] = keys
        out[f"sens{i}_bits"] = np.array([bits])
        out[f"sens{i}_mse"] = rep.mse
        out[f"sens{i}_ranking"] = rep.ranking
    out["num_sens"] = np.array([len(SENS)])
    for i, (L, d, heads, lq, frac, seed) in enumerate(SWEEP):
        rng = np.random.default_rng(seed)
        keys = kv.generate_synthetic(kv.SyntheticSpec(tokens=L, channels=d, outlier_channels=(1, 5),
                                                      outlier_gain=6.0, seed=seed))
        queries = rng.normal(0, 1, (heads, lq, d)).astype(np.float32)
        sel = kv.select_boost(kv.channel_scores(keys), frac).boosted
        out[f"sweep{i}_k"] = keys
        out[f"sweep{i}_q"] = queries
        out[f"sweep{i}_sel"] = sel
        out[f"sweep{i}_mse_sel"] = np.array([an.attention_mse(keys, queries, sel)])
        out[f"sweep{i}_mse_none"] = np.array([an.attention_mse(keys, queries, [])])
        rows = an.boost_sweep(keys, queries, [0.0, 0.0625, frac, 0.5], random_draws=3, seed=seed)
        out[f"sweep{i}_rows"] = np.array([[r.fraction, r.heuristic == "magnitude", r.mean_mse, r.max_deviation, r.runs]
                                          for r in rows])
    out["num_sweep"] = np.array([len(SWEEP)])
    rows = an.boost_sweep_experiment([0.0, 0.125, 0.25], n_seeds=3, tokens=256, channels=32,
                                     outlier_channels=(3, 17), query_tokens=32)
    out["experiment_rows"] = np.array([[r.fraction, r.heuristic == "magnitude", r.mean_mse, r.max_deviation, r.runs]
                                       for r in rows])
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()
