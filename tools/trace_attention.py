"""Per-warp timeline of one fused-attention launch (debug; run on the GPU box).

python tools/trace_attention.py [--context 32768] [--batch 16]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18643_b200 as kb  # noqa: E402
from paper_2511_18643_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--batch", type=int, default=16)
args = ap.parse_args()

cfg = kb.KittyConfig(h_kv=8, h_q=32)
dev = torch.device("cuda")
cache = kb.KittyBatchCache(cfg, args.batch, args.context + 8)
g = torch.Generator(device=dev)
g.manual_seed(0)
for b in range(args.batch):
    pass
k = torch.randn((args.batch, 8, args.context, 128), generator=g, device=dev).bfloat16()
v = torch.randn((args.batch, 8, args.context, 128), generator=g, device=dev).bfloat16()
cache.prefill(k, v)
del k, v
q = torch.randn((args.batch, 32, 128), generator=g, device=dev).bfloat16()
for _ in range(3):
    cache.attend(q)
torch.cuda.synchronize()
lib = kb.load_library()
lib.kitty_debug_attention_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
n = 148 * 2 * 4
buf = np.zeros((16384, 10), np.int64)
lib.kitty_debug_attention_trace(1, None, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cache.attend(q)
e1.record()
torch.cuda.synchronize()
lib.kitty_debug_attention_trace(0, buf.ctypes.data, 16384)
r = buf[:n]
r = r[r[:, 1] > 0]
t0 = r[:, 1].min()
start = (r[:, 1] - t0) / 1e3
end = (r[:, 2] - t0) / 1e3
print(f"launch {e0.elapsed_time(e1) * 1e3:.1f} us; warps traced {len(r)}")
print(f"warp start: min {start.min():.1f} max {start.max():.1f} us")
print(f"warp end:   min {end.min():.1f} p10 {np.percentile(end, 10):.1f} p50 {np.percentile(end, 50):.1f} p90 {np.percentile(end, 90):.1f} max {end.max():.1f} us")
print(f"fp items per warp: mean {r[:, 3].mean():.2f} max {r[:, 3].max()}; pages per warp mean {r[:, 4].mean():.1f} min {r[:, 4].min()} max {r[:, 4].max()}")
print(f"fp time per warp us: mean {r[:, 5].mean() / 1e3:.1f} max {r[:, 5].max() / 1e3:.1f}; per fp item {r[:, 5].sum() / max(1, r[:, 3].sum()) / 1e3:.2f}")
print(f"merge time per warp us: mean {r[:, 6].mean() / 1e3:.1f} max {r[:, 6].max() / 1e3:.1f}")
print(f"key-slot wait per warp us: mean {r[:, 7].mean() / 1e3:.1f} max {r[:, 7].max() / 1e3:.1f}; per page {r[:, 7].sum() / max(1, r[:, 4].sum()):.0f} ns")
busy = (end - start)
print(f"page time per warp (excl fp/merge): {((busy * 1e3 - (r[:, 5] + r[:, 6]) / 1e3) / np.maximum(r[:, 4], 1)).mean():.0f} ns")
sm = r[:, 0]
per_sm_end = np.array([end[sm == s].max() for s in np.unique(sm)])
print(f"per-SM last warp end: min {per_sm_end.min():.1f} p50 {np.median(per_sm_end):.1f} max {per_sm_end.max():.1f} us")
order = np.argsort(end)[-8:]
for i in order:
    print(f"  late warp sm {r[i, 0]} end {end[i]:.1f} fp {r[i, 3]} pages {r[i, 4]} fp_us {r[i, 5] / 1e3:.1f} merge_us {r[i, 6] / 1e3:.1f}")

# compute-only: same launch with page loads skipped (stale shared-memory pages)
lib.kitty_debug_attention_trace(3, None, 0)
cache.attend(q)
torch.cuda.synchronize()
lib.kitty_debug_attention_trace(0, buf.ctypes.data, 16384)
r = buf[:n]
r = r[r[:, 1] > 0]
t0 = r[:, 1].min()
end = (r[:, 2] - t0) / 1e3
print(f"[compute-only] warp end p50 {np.percentile(end, 50):.1f} max {end.max():.1f} us; page time per warp "
      f"{((end * 1e3 - r[:, 5] / 1e3) / np.maximum(r[:, 4], 1)).mean():.0f} ns")
