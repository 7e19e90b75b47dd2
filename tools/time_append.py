"""Time decode appends on the C2 shape, including the steps that pack a key
page (q-buffer full) or a value page (ring full): CUDA events per append."""
import sys

import torch

import paper_2511_18643_b200 as K

cfg = K.KittyConfig(s=32, r=128, g=128, d=128, h_kv=8, h_q=32, boost_fraction=0.125)
B = 16
c = K.KittyBatchCache(cfg, B, 1024)
k = torch.randn(B, 8, 1024, 128, device="cuda").bfloat16()
v = torch.randn(B, 8, 1024, 128, device="cuda").bfloat16()
c.prefill(k[:, :, :300], v[:, :, :300])
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
plain, packs = [], []
for t in range(300, 700):
    ev[0].record()
    c.append(k[:, :, t], v[:, :, t])
    ev[1].record()
    torch.cuda.synchronize()
    past = t + 1 - 32
    (packs if past % 128 == 0 or (past - 128) % 128 == 0 else plain).append(ev[0].elapsed_time(ev[1]) * 1e3)
plain.sort()
print(f"append us: plain median {plain[len(plain) // 2]:.1f}; pack steps {[round(x, 1) for x in packs]}")
