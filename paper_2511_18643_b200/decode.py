"""Multi-layer decode step over Kitty caches, with CUDA-graph replay.

A model's decode step runs, for every attention layer, ``append`` (insert the
new K/V rows, pack full q-buffers) then ``attend`` (fused dequant-attention)
-- the reference's loop body (cli.py:310-315, cache.py:107-252) for a batch
of sequences.  ``DecodeStep`` owns fixed input/output buffers so the whole
step (2 launches per layer + the split combine) is captured once into a CUDA
graph and replayed; the device reads sequence lengths from HBM, so the same
graph serves every step.
"""

from __future__ import annotations

import torch

from . import _lib
from .cache import KittyBatchCache
from .config import KittyConfig
from .pages import _stream


class DecodeStep:
    def __init__(self, cfg: KittyConfig, num_layers: int, num_seqs: int, max_tokens: int, device=None, shard=None):
        self.cfg = cfg
        self.shard = shard  # sharding.Shard this step serves (None: the whole model on one GPU)
        self.num_layers = num_layers
        self.num_seqs = num_seqs
        self.max_tokens = max_tokens
        self.layers = [KittyBatchCache(cfg, num_seqs, max_tokens, device) for _ in range(num_layers)]
        dev = self.layers[0].device
        self.device = dev
        bf = torch.bfloat16
        # the step's inputs in one flat buffer (k | v | q): a caller refreshes
        # them with a single copy per step
        nk = num_layers * num_seqs * cfg.h_kv * cfg.d
        nq = num_layers * num_seqs * cfg.h_q * cfg.d
        self.inputs = torch.zeros(2 * nk + nq, dtype=bf, device=dev)
        self.k_in = self.inputs[:nk].view(num_layers, num_seqs, cfg.h_kv, cfg.d)
        self.v_in = self.inputs[nk:2 * nk].view(num_layers, num_seqs, cfg.h_kv, cfg.d)
        self.q_in = self.inputs[2 * nk:].view(num_layers, num_seqs, cfg.h_q, cfg.d)
        self.out = torch.zeros((num_layers, num_seqs, cfg.h_q, cfg.d), dtype=bf, device=dev)
        # one workspace shared by the layers (they run back to back on one stream)
        self.ws = self.layers[0].workspace(max_tokens)
        self.graph = None
        self.lib = _lib.load_library()

    @classmethod
    def for_shard(cls, cfg: KittyConfig, shard, num_layers: int, max_tokens: int, device=None) -> "DecodeStep":
        """The decode step of one rank of a multi-GPU partition (sharding.py):
        its requests and KV heads of the model config ``cfg``."""
        return cls(shard.local_config(cfg), num_layers, shard.num_seqs, max_tokens, device, shard)

    # bytes moved per step by the inputs / outputs (for the e2e host copies)
    def input_bytes(self) -> int:
        return self.inputs.numel() * self.inputs.element_size()

    def pack_inputs(self, k, v, q) -> torch.Tensor:
        """k / v [layers, B, h_kv, D], q [layers, B, h_q, D] -> one flat tensor
        laid out like ``inputs`` (leading batch dimensions of k, v, q kept)."""
        lead = k.shape[:-4]
        return torch.cat([k.reshape(*lead, -1), v.reshape(*lead, -1), q.reshape(*lead, -1)], dim=-1)

    def output_bytes(self) -> int:
        return self.out.numel() * self.out.element_size()

    def launches_per_step(self) -> int:
        return self.num_layers * (1 + self.attention_launches())

    def attention_launches(self) -> int:
        # mma.sync path (default): fp-token chunks + pages + split-KV merge;
        # the tcgen05 path (kitty_debug_select_attention) launches 2
        return 3

    def fast_path(self) -> bool:
        c = self.cfg
        return c.d == 128 and c.g == 128 and c.group_size in (1, 2, 4, 8) and c.d_boost <= 32

    def _launch(self):
        lib, st = self.lib, _stream()
        for l, cache in enumerate(self.layers):
            _lib.check(lib.kitty_append(cache._desc_ref, self.k_in[l].data_ptr(), self.v_in[l].data_ptr(), st), "append")
            _lib.check(lib.kitty_decode_attention(cache._desc_ref, self.q_in[l].data_ptr(), self.out[l].data_ptr(),
                                                  _lib.KITTY_BF16, self.max_tokens, self.ws.data_ptr(),
                                                  self.ws.numel(), st), "attend")

    def step(self):
        """One eager decode step over all layers."""
        if max(self.layers[0].lengths) + 1 > self.max_tokens:
            raise ValueError("decode step past the allocated context")
        # every layer holds the same lengths: the pack mirror is computed once per step
        packs = self.layers[0].append_packs()
        need = self.layers[0].append_page_need(packs)
        if need[0] or need[1]:  # the pools are sized for max_tokens: never short, but checked
            if any(need[0] > c.free_pages[0] or need[1] > c.free_pages[1] for c in self.layers):
                raise ValueError("decode step would exhaust a layer's page pool")
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch()
        for cache in self.layers:
            cache.advance_host(need, packs)

    def capture(self):
        """Capture one step into a CUDA graph (does not advance the state)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            # the capture records launches only; lengths are read on device at replay
            with torch.cuda.graph(g, stream=s):
                self._launch()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        for cache in self.layers:  # the graph holds their buffer addresses from now on
            cache.captured = True
        return g

    def attention_only(self, layer: int):
        cache = self.layers[layer]
        _lib.check(self.lib.kitty_decode_attention(cache._desc_ref, self.q_in[layer].data_ptr(), self.out[layer].data_ptr(),
                                                   _lib.KITTY_BF16, self.max_tokens, self.ws.data_ptr(), self.ws.numel(),
                                                   _stream()), "attend")

    def append_only(self, layer: int):
        cache = self.layers[layer]
        _lib.check(self.lib.kitty_append(cache._desc_ref, self.k_in[layer].data_ptr(), self.v_in[layer].data_ptr(),
                                         _stream()), "append")
