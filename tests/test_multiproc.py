"""N>1 path on CPU: world_size-2 gloo processes, each owning a request (or KV
head) shard of a decode step; the optional output all_gather must rebuild the
single-process result exactly.  The per-rank compute here is the CPU oracle
(the GPU kernel is covered by the -m gpu tests); what is under test is the
partition and gather logic the multi-GPU bench uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_18643_b200 import sharding
from paper_2511_18643_b200.config import KittyConfig
from oracle import kitty_oracle as ko

CFG = dict(s=4, r=8, g=8, d=8, h_kv=4, h_q=8, boost_fraction=0.25)
BATCH, N = 4, 45


def _inputs():
    rng = np.random.default_rng(123)
    keys = rng.normal(0, 1, (BATCH, CFG["h_kv"], N, CFG["d"])).astype(np.float32)
    values = rng.normal(0, 1, (BATCH, CFG["h_kv"], N, CFG["d"])).astype(np.float32)
    q = rng.normal(0, 1, (BATCH, CFG["h_q"], CFG["d"])).astype(np.float32)
    return keys, values, q


def _attend(keys, values, q, h_kv, h_q):
    c = dict(CFG, h_kv=h_kv, h_q=h_q)
    out = np.empty((keys.shape[0], h_q, c["d"]), np.float32)
    for b in range(keys.shape[0]):
        st = ko.OracleCache(c["s"], c["r"], c["g"], c["d"], h_kv, h_q, c["boost_fraction"])
        st.prefill(keys[b], values[b])
        out[b] = st.attend(q[b])
    return out


def _worker(rank, world, port, mode, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    keys, values, q = _inputs()
    cfg = KittyConfig(**CFG)
    sh = sharding.make_shard(mode, BATCH, cfg.h_kv, world, rank)
    local_cfg = sh.local_config(cfg)  # the shape DecodeStep.for_shard allocates on this rank
    assert local_cfg.group_size == cfg.group_size and local_cfg.d_boost == cfg.d_boost
    k, v, qq = sh.select_kv(keys, cfg), sh.select_kv(values, cfg), sh.select_q(q, cfg)
    assert k.shape[:2] == (sh.num_seqs, local_cfg.h_kv) and qq.shape[:2] == (sh.num_seqs, local_cfg.h_q)
    local = _attend(k, v, qq, local_cfg.h_kv, local_cfg.h_q)
    full = sharding.gather_outputs(torch.from_numpy(local), mode)
    if rank == 0:
        result.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["request", "kv_head"])
def test_two_rank_shards_rebuild_full_step(mode):
    ctx = mp.get_context("spawn")
    result = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, result)) for r in range(2)]
    for p in procs:
        p.start()
    got = result.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    keys, values, q = _inputs()
    want = _attend(keys, values, q, CFG["h_kv"], CFG["h_q"])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shards_cover_every_unit_once(world):
    # every (sequence, KV head) unit of the C5 shape lands on exactly one rank
    cfg = KittyConfig(h_kv=8, h_q=64)
    for mode in ("request", "kv_head"):
        seen = np.zeros((16, cfg.h_kv), int)
        for r in range(world):
            sh = sharding.make_shard(mode, 16, cfg.h_kv, world, r)
            seen[sh.seq_begin:sh.seq_end, sh.kv_begin:sh.kv_end] += 1
            assert sh.local_config(cfg).h_q == sh.num_kv_heads * 8
        assert (seen == 1).all()
