"""GPU parity of the attention launch variants that the A/B knobs select
(kitty_attention_fast.cu reads them once per process, so each runs in a
subprocess): the launch order (fp grid first / page grid first), the
warp-specialised page kernel at every GQA group (the default only at group 8),
programmatic dependent launch off, and the CTA-per-chunk full-precision
kernel (with and without the shared page / key-tile layout) where the
warp-per-chunk one is the default.  Every variant must give the same
answer as the oracle within the attention bar (max-abs 1e-2), on a ragged
batch with a short and a long (> 128 partial slots) unit."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch
import paper_2511_18643_b200 as kb
from oracle import kitty_oracle as ko
kb.load_library()

def bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()

worst = 0.0
for group in (1, 2, 4, 8):
    rng = np.random.default_rng(group)
    b, h_kv = 2, 2
    lens = [700, 20000]
    n = max(lens)
    cfg = kb.KittyConfig(h_kv=h_kv, h_q=h_kv * group)
    k = rng.normal(0, 1, (b, h_kv, n, 128)).astype(np.float32)
    k[..., rng.choice(128, 16, replace=False)] *= 8
    k, v = bf16(k), bf16(rng.normal(0, 1, (b, h_kv, n, 128)))
    cache = kb.KittyBatchCache(cfg, b, n + 2)
    cache.prefill(torch.from_numpy(k), torch.from_numpy(v), lengths=lens)
    q = bf16(rng.normal(0, 1, (b, h_kv * group, 128)))
    for rep in range(2):  # the second call reuses the workspace the first left
        out = cache.attend(torch.from_numpy(q).cuda(), out_dtype=torch.float32).cpu().numpy()
    cache.check()
    for bi, ln in enumerate(lens):
        for h in range(h_kv):
            kf, vf, _, _ = ko.bulk_unit_state(k[bi, h, :ln], v[bi, h, :ln], 32, 128, 128, 0.125, metadata16=True)
            qg = q[bi, h * group:(h + 1) * group]
            worst = max(worst, float(np.max(np.abs(out[bi, h * group:(h + 1) * group] - ko.attend_rows(kf, vf, qg)))))
print("WORST", worst)
"""


@pytest.mark.parametrize("env", [{"KITTY_FPFIRST": "1"}, {"KITTY_FPFIRST": "0"}, {"KITTY_WS": "1"},
                                 {"KITTY_WS": "0"}, {"KITTY_PDL": "0"}, {"KITTY_WS": "1", "KITTY_FPFIRST": "0"},
                                 {"KITTY_FPWARP": "0"}, {"KITTY_FPWARP": "0", "KITTY_FPUNION": "0"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_launch_variant_matches_oracle(cuda, env):
    full = dict(os.environ, **env)
    full["PYTHONPATH"] = ROOT + os.pathsep + full.get("PYTHONPATH", "")
    res = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=full, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    worst = float(res.stdout.strip().splitlines()[-1].split()[1])
    assert worst <= 1e-2, (env, worst)
