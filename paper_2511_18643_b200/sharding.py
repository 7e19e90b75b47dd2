"""Multi-GPU partitioning of the decode hot path.

Units (sequence, KV head, layer) are independent: attention has no cross-unit
reduction, so the path shards with NO collective on the data path.  One
process per GPU; each rank owns either a contiguous slice of the request batch
(C2-C4: weak scaling) or a contiguous slice of the KV heads with their query
groups for every request (C5: strong scaling, the 70B cache does not fit one
GPU).  A rank's cache is an ordinary ``KittyBatchCache`` / ``DecodeStep`` of
its local shape (``Shard.local_config``); its inputs are the slices
``select_kv`` / ``select_q`` cut from the full step's tensors.  The only
optional collective is an all_gather of the bf16 outputs, kept off the timed
path (``gather_outputs``).
"""

from __future__ import annotations

from dataclasses import dataclass

from .config import KittyConfig


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    seq_begin: int
    seq_end: int
    kv_begin: int
    kv_end: int
    mode: str = "request"

    @property
    def num_seqs(self) -> int:
        return self.seq_end - self.seq_begin

    @property
    def num_kv_heads(self) -> int:
        return self.kv_end - self.kv_begin

    def local_config(self, cfg: KittyConfig) -> KittyConfig:
        """The cache shape this rank holds: its KV heads and their query groups
        (cache.py:240 maps query head i to KV head i // group)."""
        g = cfg.group_size
        return KittyConfig(s=cfg.s, r=cfg.r, g=cfg.g, d=cfg.d, h_kv=self.num_kv_heads, h_q=self.num_kv_heads * g,
                           key_bits=cfg.key_bits, value_bits=cfg.value_bits, boost_fraction=cfg.boost_fraction,
                           heuristic=cfg.heuristic, heuristic_seed=cfg.heuristic_seed)

    def select_kv(self, t, cfg: KittyConfig):
        """This rank's part of a [B, h_kv, ...] tensor (new K / V rows, prompts)."""
        return t[self.seq_begin:self.seq_end, self.kv_begin:self.kv_end]

    def select_q(self, t, cfg: KittyConfig):
        """This rank's part of a [B, h_q, ...] tensor (queries, outputs)."""
        g = cfg.group_size
        return t[self.seq_begin:self.seq_end, self.kv_begin * g:self.kv_end * g]


def _split(n: int, world: int, rank: int) -> tuple[int, int]:
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_by_request(batch: int, h_kv: int, world: int, rank: int) -> Shard:
    """Contiguous request slice per rank; every rank keeps all KV heads."""
    if not 0 <= rank < world:
        raise ValueError("rank outside world")
    b0, b1 = _split(batch, world, rank)
    return Shard(rank, world, b0, b1, 0, h_kv, "request")


def shard_by_kv_head(batch: int, h_kv: int, world: int, rank: int) -> Shard:
    """Contiguous KV-head slice per rank (with its h_q / h_kv query heads);
    every rank keeps all requests.  Needs h_kv % world == 0 for balance."""
    if not 0 <= rank < world:
        raise ValueError("rank outside world")
    h0, h1 = _split(h_kv, world, rank)
    return Shard(rank, world, 0, batch, h0, h1, "kv_head")


def make_shard(mode: str, batch: int, h_kv: int, world: int, rank: int) -> Shard:
    if mode == "request":
        return shard_by_request(batch, h_kv, world, rank)
    if mode == "kv_head":
        return shard_by_kv_head(batch, h_kv, world, rank)
    raise ValueError(f"unknown shard mode {mode!r}")


def gather_outputs(local_out, mode: str, group=None):
    """Optional all_gather of per-rank outputs into the full batch (off the
    timed path).  ``mode`` "request": local [B/world, h_q, d] -> [B, h_q, d];
    "kv_head": local [B, h_q/world, d] -> [B, h_q, d].  Shards must be
    balanced (all_gather needs equal shapes)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    local_out = local_out.contiguous()
    parts = [torch.empty_like(local_out) for _ in range(world)]
    dist.all_gather(parts, local_out, group=group)
    return torch.cat(parts, dim=0 if mode == "request" else 1)
