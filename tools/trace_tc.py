"""Event timeline of CTA 0 of one tc attention launch (debug; run on the GPU box).

python tools/trace_tc.py [--context 32768] [--batch 16]
Fields per page: 0 TMA issue, 1 WG-A full, 2 WG-A sfree, 3 WG-A kready, 4 MMA QK,
5 WG-B sfull, 6 WG-B pready, 7 MMA PV, 8 WG-C vready, 9 WG-C ofull.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18643_b200 as kb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--rows", type=int, default=40)
args = ap.parse_args()

cfg = kb.KittyConfig(h_kv=8, h_q=32)
dev = torch.device("cuda")
cache = kb.KittyBatchCache(cfg, args.batch, args.context + 8)
g = torch.Generator(device=dev)
g.manual_seed(0)
k = torch.randn((args.batch, 8, args.context, 128), generator=g, device=dev).bfloat16()
v = torch.randn((args.batch, 8, args.context, 128), generator=g, device=dev).bfloat16()
cache.prefill(k, v)
del k, v
q = torch.randn((args.batch, 32, 128), generator=g, device=dev).bfloat16()
for _ in range(3):
    cache.attend(q)
torch.cuda.synchronize()
lib = kb.load_library()
lib.kitty_debug_tc_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
lib.kitty_debug_select_attention(1)
buf = np.zeros((512, 24), np.int64)
lib.kitty_debug_tc_trace(1, None, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cache.attend(q)
e1.record()
torch.cuda.synchronize()
lib.kitty_debug_tc_trace(0, buf.ctypes.data, 512)
print(f"launch (attention + combine) {e0.elapsed_time(e1) * 1e3:.1f} us")
valid = buf[:, 0] > 0
n = int(valid.sum())
t0 = buf[valid][:, 0].min()
r = np.where(buf > 0, buf - t0, -1)
print(f"CTA 0 pages: {n}, last event at {r.max() / 1e3:.1f} us")
names = ["tma", "A.full", "A.sfree", "A.kready", "mma.qk", "B.sfull", "B.pready", "mma.pv", "C.vready", "C.ofull", "A.bound", "A.conv", "A.brow", "A.fence", "B.tmld", "B.max", "B.vready", "B.vfree", "B.sts", "B.ring", "B.fence"]
print("page " + " ".join(f"{x:>9s}" for x in names[:16]))
for i in list(range(min(args.rows, n))) + list(range(max(args.rows, n - 10), n)):
    print(f"{i:4d} " + " ".join(f"{x / 1e3:9.2f}" for x in r[i][:16]))
d = np.diff(r[:n], axis=0)
print("median per-page delta (us): " + " ".join(f"{np.median(d[:, f]) / 1e3:.3f}" for f in range(21)))
lat = lambda a, b: np.median(r[:n, b] - r[:n, a]) / 1e3
print(f"median latencies (us): tma->A.full {lat(0, 1):.2f}  A.full->A.kready {lat(1, 3):.2f}  A.kready->qk {lat(3, 4):.2f}  "
      f"qk->B.sfull {lat(4, 5):.2f}  B.sfull->pready {lat(5, 6):.2f}  pready->pv {lat(6, 7):.2f}  pv->C.ofull {lat(7, 9):.2f}")
print(f"WG-A: sfree->bound {lat(2, 10):.3f} bound->conv-done {lat(10, 11):.3f} conv->brow-done {lat(11, 12):.3f} brow->zsum-done {lat(12, 13):.3f} zsum->kready {lat(13, 3):.3f}")
print(f"WG-B: sfull->tmld {lat(5, 14):.3f} tmld->max {lat(14, 15):.3f} max->vready {lat(15, 16):.3f} vready->vfree {lat(16, 17):.3f} vfree->sts {lat(17, 18):.3f} sts->ring {lat(18, 19):.3f} ring->fence {lat(19, 20):.3f} fence->pready {lat(20, 6):.3f}")
