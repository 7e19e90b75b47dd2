"""The library's A/B knobs (read once when it loads) must not change results:
KITTY_PDL=0 serialises the page / fp-token / merge grids, KITTY_FAST_PACK=0
keeps prefill on the generic packer.  Each setting runs in a subprocess on the
same seeded inputs; outputs and page bytes are compared with this process
(defaults)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2511_18643_b200 as kb
torch.manual_seed(0)
cfg = kb.KittyConfig(h_kv=2, h_q=8)
lens = [1300, 700, 2100]
k = torch.randn(3, 2, 2100, 128).bfloat16()
v = torch.randn(3, 2, 2100, 128).bfloat16()
q = torch.randn(3, 8, 128).bfloat16()
c = kb.KittyBatchCache(cfg, 3, 2200)
c.prefill(k, v, lengths=lens)
out = c.attend(q.cuda()).float().cpu().numpy()
c.check()
pages = np.frombuffer(b"".join(b"".join(kp) + b"".join(vp) for kp, vp in (c.export_pages(b, h) for b in range(3) for h in range(2))), np.uint8)
np.savez({path!r}, out=out, pages=pages)
"""


def _run(tmp_path, name, env_extra):
    path = str(tmp_path / f"{name}.npz")
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, path=path)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return dict(np.load(path))


@pytest.mark.gpu
def test_knobs_do_not_change_results(cuda, tmp_path):
    base = _run(tmp_path, "base", {})
    serial = _run(tmp_path, "serial", {"KITTY_PDL": "0"})
    generic = _run(tmp_path, "generic", {"KITTY_FAST_PACK": "0"})
    # identical launches in a different order / overlap: identical bits
    assert np.array_equal(base["out"], serial["out"])
    assert np.array_equal(base["pages"], serial["pages"])
    # the bulk packer and the generic packer write the same page bytes
    assert np.array_equal(base["pages"], generic["pages"])
    assert np.array_equal(base["out"], generic["out"])
