#!/usr/bin/env python3
"""Decode-attention benchmark of the Kitty hot path on B200.

Workload (BASELINE.json configs[1], fits one GPU): LLaMA3-8B attention shape
-- 32 layers, GQA 32 q / 8 kv heads, head_dim 128 -- batch 16, 32K context,
Kitty 2-bit K/V + 12.5 % boosted key channels.  One step = for every layer:
append one token (insert + pack when a q-buffer fills) and attend over the
whole cache with pages dequantised on the fly.  Metric: decode tokens/s
(= sequences / step time) and achieved HBM GB/s of the attention kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kitty|reference]
                    [--config c1..c5] [--shard request|kv_head]

N > 1: one process per GPU (re-executed under torch.distributed.run when
WORLD_SIZE is unset).  The units (sequence, KV head, layer) are independent,
so ranks share no data-path collective:
  * --shard request (default; C1-C4): every rank owns its own batch (weak
    scaling, global batch = batch x N);
  * --shard kv_head (default for C5): every rank owns h_kv / N KV heads and
    their query groups for the whole global batch (strong scaling).  An
    NCCL all_gather of the outputs is timed separately, off the step.
The reference arm (--impl reference) times the reference implementation
itself (`kittykv`, installed into baseline/_ref) on this host's cores, on one
(sequence, layer) slice of the same workload, extrapolated to the step; the
numpy restatement in oracle/ stands in only if kittykv cannot be imported.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn tokens/sec and achieved HBM GB/s (% of roofline) at 1/2/4/8 B200"
CONFIGS = {
    # name: (layers, batch, context, h_kv, h_q, boost_fraction, default shard, description)
    # batch is per GPU for request sharding, global for KV-head sharding
    "c1": (1, 1, 4096, 8, 32, 0.125, "request", "single-layer synthetic: batch 1, 8 kv / 32 q heads, d 128, 4K context"),
    "c2": (32, 16, 32768, 8, 32, 0.125, "request", "LLaMA3-8B attention shape (32 layers, GQA 32q/8kv, d=128), batch 16, 32K context"),
    "c3": (36, 64, 8192, 8, 32, 0.125, "request", "Qwen3-8B attention shape (36 layers, GQA 32q/8kv, d=128), batch 64, 8K context"),
    "c4": (32, 1, 131072, 8, 32, 0.125, "request", "LLaMA3-8B long context 128K, 1 request per GPU (batch 8 over 8 GPUs)"),
    "c5": (80, 256, 16384, 8, 64, 0.125, "kv_head", "LLaMA3-70B attention shape (80 layers, GQA 64q/8kv), batch 256, 16K context, KV heads sharded"),
}
OUTLIERS = 16  # outlier key channels (x8), SyntheticSpec-style (tensor_io.py:89-124)
HBM_BUDGET = 120e9  # bytes of cache per GPU the C5 batch is fitted to (prefill temporaries need the rest)


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload (shared by both arms, so their `config` dicts are identical)
# ---------------------------------------------------------------------------


def workload(args, world: int) -> dict:
    layers, batch, ctx, h_kv, h_q, frac, shard, desc = CONFIGS[args.config]
    shard = args.shard or shard
    layers = args.layers or layers
    ctx = args.context or ctx
    frac = frac if args.boost is None else args.boost
    if shard == "kv_head":
        if h_kv % world:
            raise SystemExit(f"--shard kv_head needs h_kv ({h_kv}) divisible by the GPU count ({world})")
        h_kv_l, h_q_l = h_kv // world, h_q // world
        if args.batch:
            gbatch = args.batch
        else:  # the global batch, capped to what fits the per-GPU cache budget
            from paper_2511_18643_b200.analysis import algorithmic_bytes_per_unit
            from paper_2511_18643_b200.config import KittyConfig

            unit = algorithmic_bytes_per_unit(KittyConfig(h_kv=h_kv, h_q=h_q, boost_fraction=frac), ctx)
            per_seq = layers * h_kv_l * (unit + 2 * 128 * (2 * 32 + 128 + 256))  # + sinks, q-buffer, value ring
            gbatch = min(batch, max(8, int(HBM_BUDGET // per_seq) // 8 * 8))
        batch_l = gbatch
    else:
        h_kv_l, h_q_l = h_kv, h_q
        batch_l = args.batch or batch
        gbatch = batch_l * world
    return dict(config=args.config, workload=desc, layers=layers, global_batch=gbatch, batch_per_gpu=batch_l,
                context=ctx, h_kv=h_kv, h_q=h_q, h_kv_per_gpu=h_kv_l, h_q_per_gpu=h_q_l, head_dim=128,
                boost_fraction=frac, shard=shard, n_gpus=world,
                parallelism=(f"KV heads sharded x{world} ({h_kv_l} kv / {h_q_l} q heads per GPU, all requests)"
                             if shard == "kv_head" else f"requests sharded x{world} ({batch_l} per GPU)"))


# ---------------------------------------------------------------------------
# Kitty (GPU) arm
# ---------------------------------------------------------------------------


def run_kitty(args):
    import torch
    import torch.distributed as dist

    import paper_2511_18643_b200 as kb
    from paper_2511_18643_b200 import sharding
    from paper_2511_18643_b200.decode import DecodeStep

    rank, world, local = _env_rank()
    if world > 1:
        # one process per GPU over NCCL; --dist-backend gloo lets N ranks share one
        # GPU (a smoke test of the N > 1 path on a single-GPU box)
        torch.cuda.set_device(local % torch.cuda.device_count())
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", torch.cuda.current_device())
    rdev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # reductions of timings
    wl = workload(args, world)
    layers, ctx = wl["layers"], wl["context"]
    model_cfg = kb.KittyConfig(h_kv=wl["h_kv"], h_q=wl["h_q"], boost_fraction=wl["boost_fraction"])
    shard = sharding.make_shard(wl["shard"], wl["global_batch"], wl["h_kv"], world, rank)
    steps, warmup = args.steps, args.warmup
    max_tokens = ctx + warmup + 2 * steps + 8
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    step = DecodeStep.for_shard(model_cfg, shard, layers, max_tokens, dev)
    cfg, batch = step.cfg, step.num_seqs

    # -- synthetic prefill (not timed): K ~ N(0,1) with x8 outlier channels, V ~ N(0,1), bf16.
    # The raw rows of the sampled parity units (layer 0) are kept on the host.
    outl = torch.randperm(cfg.d, generator=gen, device=dev)[:OUTLIERS]
    gain = torch.ones(cfg.d, device=dev)
    gain[outl] = 8.0
    sample_units = sorted({(0, 0), (batch - 1, cfg.h_kv - 1)})
    kept = {}
    t0 = time.time()
    chunk = max(1, min(batch, (1 << 31) // (cfg.h_kv * ctx * cfg.d * 2)))
    for li, cache in enumerate(step.layers):
        for b0 in range(0, batch, chunk):
            nb = min(chunk, batch - b0)
            k = (torch.randn((nb, cfg.h_kv, ctx, cfg.d), generator=gen, device=dev) * gain).bfloat16()
            v = torch.randn((nb, cfg.h_kv, ctx, cfg.d), generator=gen, device=dev).bfloat16()
            if li == 0:
                for (b, h) in sample_units:
                    if b0 <= b < b0 + nb:
                        kept[(b, h)] = (k[b - b0, h].float().cpu(), v[b - b0, h].float().cpu())
            cache.prefill_range(b0, nb, k, v)
            del k, v
    torch.cuda.synchronize()
    prefill_s = time.time() - t0
    for c in step.layers:
        c.check()

    # per-step inputs resident in HBM (a fresh token per step and layer)
    n_in = warmup + steps
    ks = (torch.randn((n_in, layers, batch, cfg.h_kv, cfg.d), generator=gen, device=dev) * gain).bfloat16()
    vs = torch.randn((n_in, layers, batch, cfg.h_kv, cfg.d), generator=gen, device=dev).bfloat16()
    qs = torch.randn((n_in, layers, batch, cfg.h_q, cfg.d), generator=gen, device=dev).bfloat16()

    use_graph = not args.no_graph
    if use_graph:
        step.capture()

    xs = step.pack_inputs(ks, vs, qs)  # [n_in, k | v | q] resident in HBM
    nk = ks[0].numel()  # ks / vs / qs become views of xs (one copy of the inputs in HBM)
    ks, vs, qs = (xs[:, :nk].view(ks.shape), xs[:, nk:2 * nk].view(vs.shape), xs[:, 2 * nk:].view(qs.shape))

    def one(i):
        step.inputs.copy_(xs[i])
        step.step()

    for i in range(warmup):
        one(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall0 = time.time()
    e0.record()
    for i in range(warmup, warmup + steps):
        one(i)
    e1.record()
    torch.cuda.synchronize()
    wall = time.time() - wall0
    ms_local = e0.elapsed_time(e1)
    ms = _max_over_ranks(ms_local, world, rdev)
    clk = clocks.stop()
    ms_per_step = ms / steps
    for c in step.layers:
        c.check()

    # -- parity: the last step's outputs of the sampled units (layer 0) against
    # the oracle's attend over the same rows (prefill + every appended token)
    parity = None
    if not args.no_parity:
        parity = _gather_parity(_parity(cfg, step, kept, ks, vs, qs, n_in, sample_units), world, rdev)

    # -- attention kernel alone (pages + fp tokens + merge of every layer), captured
    # in one CUDA graph and replayed between CUDA events on the launching stream, so
    # the per-launch time is device time without host launch overhead
    ga = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        with torch.cuda.graph(ga, stream=cs):
            for l in range(layers):
                step.attention_only(l)
    torch.cuda.current_stream().wait_stream(cs)
    reps = max(2, 64 // layers)
    for _ in range(2):
        ga.replay()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a0.record()
    for _ in range(reps):
        ga.replay()
    a1.record()
    torch.cuda.synchronize()
    attn_avg_ms = a0.elapsed_time(a1) / (reps * layers)
    n_now = step.layers[0].lengths[0]
    bytes_per_launch = batch * cfg.h_kv * kb.algorithmic_bytes_per_unit(cfg, n_now)
    peak, peak_kind = _measured_peaks()
    achieved = bytes_per_launch / (attn_avg_ms * 1e-3) / 1e9

    # -- the KV-head split's optional collective: all_gather of one layer's
    # outputs, timed on its own (not part of the step)
    collective = None
    if world > 1 and wl["shard"] == "kv_head" and args.dist_backend == "nccl":
        o = step.out[0].contiguous()
        parts = [torch.empty_like(o) for _ in range(world)]
        for _ in range(3):
            dist.all_gather(parts, o)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        c0.record()
        for _ in range(10):
            dist.all_gather(parts, o)
        c1.record()
        torch.cuda.synchronize()
        collective = {"op": "nccl all_gather of one layer's outputs [B, h_q, d] bf16 (off the timed step)",
                      "bytes_per_rank": o.numel() * o.element_size(),
                      "ms": round(_max_over_ranks(c0.elapsed_time(c1) / 10, world, rdev), 4),
                      "nccl_nranks": world}

    e2e_ms = _e2e(step, ks, vs, qs, warmup, steps, world, rdev)
    e2e_tps = wl["global_batch"] / (e2e_ms / steps * 1e-3)
    bytes_step = layers * bytes_per_launch
    tps = wl["global_batch"] / (ms_per_step * 1e-3)
    per_rank = _all_values(batch / (ms_local / steps * 1e-3), world, rdev)
    line = {
        "metric": METRIC,
        "value": round(tps, 2),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if wl["shard"] == "kv_head" else "weak",
        "vs_baseline": None,
        "dtype": "u8 2-bit codes -> fp16 MMA / fp32 accumulate (bf16 in/out)",
        "data": "synthetic: K ~ N(0,1) with 16 outlier channels x8, V,q ~ N(0,1), rounded to bf16; random-init, no checkpoint",
        "config": {**wl, "cuda_graph": use_graph,
                   "l2": f"working set {bytes_step / 1e9:.2f} GB/step/GPU >> 126 MB L2 (no flush needed)"},
        "prefill_s": round(prefill_s, 2),
        "hbm_gbs_step": round(bytes_step / (ms_per_step * 1e-3) / 1e9, 1),
        "roofline": {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": _ncu_traffic(args.config),
            "peak_kind": peak_kind, "kernel": "kitty decode attention (per layer launch: pages + fp tokens + merge)",
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(attn_avg_ms, 4),
            "launch_timing": f"graph of {layers} attention launches x {reps} replays, CUDA events",
            "frac_of_8TBs": round(achieved / 8000.0, 4),
        },
        "e2e": {
            "value": round(e2e_tps, 2), "unit": "tokens/s",
            "h2d_bytes_per_step": step.input_bytes(), "d2h_bytes_per_step": step.output_bytes(),
            "steps": steps,
            "copies": "pinned host <-> device every step (H2D of k/v/q, D2H of the outputs), "
                      "pipelined on a copy stream when a step moves > 1 MB",
        },
        "gpu_launches": steps * step.launches_per_step(),
        "clocks": clk,
        "wall_s_timed": round(wall, 3),
        "parity": parity,
    }
    if world > 1:
        line["per_rank_tokens_per_s"] = [round(x, 2) for x in per_rank]
        line["dist_backend"] = args.dist_backend
        line["nccl_nranks"] = world if args.dist_backend == "nccl" else 0
        line["collective"] = collective
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(wl, n_steps=1, warmup=0)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "extrapolated")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _max_over_ranks(x: float, world: int, dev) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _all_values(x: float, world: int, dev) -> list:
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device=dev)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return [float(p.item()) for p in parts]


def _parity(cfg, step, kept, ks, vs, qs, n_in, units):
    """Max-abs error of the last step's layer-0 outputs of the sampled units
    against the oracle (oracle/kitty_oracle.py, the checker; f16 page metadata
    as stored) over the same rows: the prefill plus every appended token."""
    import numpy as np

    from oracle import kitty_oracle as ko

    g = cfg.group_size
    out = step.out[0].float().cpu().numpy()
    worst, t0, n = 0.0, time.time(), 0
    for (b, h) in units:
        k0, v0 = kept[(b, h)]
        kk = np.concatenate([k0.numpy(), ks[:n_in, 0, b, h].float().cpu().numpy()])
        vv = np.concatenate([v0.numpy(), vs[:n_in, 0, b, h].float().cpu().numpy()])
        n = kk.shape[0]
        kf, vf, _, _ = ko.bulk_unit_state(kk, vv, cfg.s, cfg.r, cfg.g, cfg.boost_fraction, metadata16=True)
        want = ko.attend_rows(kf, vf, qs[n_in - 1, 0, b, h * g:(h + 1) * g].float().cpu().numpy())
        worst = max(worst, float(np.max(np.abs(out[b, h * g:(h + 1) * g] - want))))
    return {"max_abs": worst, "tol": 1e-2, "ok": worst <= 1e-2,
            "units": [f"layer 0 seq {b} kv-head {h}" for b, h in units],
            "tokens": n, "check_s": round(time.time() - t0, 1),
            "against": "oracle attend over the same rows (last timed step, bf16 output)"}


def _gather_parity(p, world, dev):
    if world == 1:
        return p
    worst = _max_over_ranks(p["max_abs"], world, dev)
    return {**p, "max_abs": worst, "ok": worst <= p["tol"], "units": f"{len(p['units'])} per rank x {world} ranks"}


def _e2e(step, ks, vs, qs, warmup, steps, world, dev) -> float:
    """The same steps through the public API with host buffers: every step copies
    its inputs from pinned host memory and its outputs back, inside the timed
    region.  Copies are pipelined as a serving loop would: step i + 1's inputs
    go host -> device staging on a copy stream while step i computes, step i's
    outputs are read back during step i + 1 (the last read-back included)."""
    import torch
    import torch.distributed as dist

    host_x = step.pack_inputs(ks[warmup:], vs[warmup:], qs[warmup:]).cpu().pin_memory()
    host_out = [torch.empty(step.out.shape, dtype=step.out.dtype).pin_memory() for _ in range(steps)]
    st_in = [torch.empty_like(step.inputs) for _ in range(2)]
    st_out = [torch.empty_like(step.out) for _ in range(2)]
    ev = lambda: torch.cuda.Event()
    in_ready, in_free, out_ready, out_free = [ev(), ev()], [ev(), ev()], [ev(), ev()], [ev(), ev()]
    main, cp = torch.cuda.current_stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    cp.wait_stream(main)
    # tiny steps (C1: 12 KB in) are host-bound: staging and events cost more than
    # the copies they hide, so those copy straight through on the compute stream
    pipelined = step.input_bytes() > (1 << 20)

    def h2d(i):
        with torch.cuda.stream(cp):
            if i >= 2:
                cp.wait_event(in_free[i % 2])
            st_in[i % 2].copy_(host_x[i], non_blocking=True)
            in_ready[i % 2].record(cp)

    if not pipelined:
        for i in range(steps):
            step.inputs.copy_(host_x[i], non_blocking=True)
            step.step()
            host_out[i].copy_(step.out, non_blocking=True)
    else:
        h2d(0)
        for i in range(steps):
            if i + 1 < steps:
                h2d(i + 1)
            main.wait_event(in_ready[i % 2])
            step.inputs.copy_(st_in[i % 2])
            in_free[i % 2].record(main)
            step.step()
            if i >= 2:
                main.wait_event(out_free[i % 2])
            st_out[i % 2].copy_(step.out)
            out_ready[i % 2].record(main)
            with torch.cuda.stream(cp):
                cp.wait_event(out_ready[i % 2])
                host_out[i].copy_(st_out[i % 2], non_blocking=True)
                out_free[i % 2].record(cp)
        main.wait_stream(cp)
    e3.record()
    torch.cuda.synchronize()
    assert all(torch.isfinite(h.float()).all() for h in host_out)
    return _max_over_ranks(e2.elapsed_time(e3), world, dev)


def _ncu_traffic(config):
    """DRAM bytes per attention launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU reference (the reference implementation itself on the host cores)
# ---------------------------------------------------------------------------


def _reference_module():
    """kittykv from baseline/_ref (the unmodified reference, pip-installed there);
    None when it is not importable (then the oracle port stands in)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import kittykv  # noqa: F401

        return kittykv
    except Exception:
        return None


def cpu_reference(wl: dict, n_steps: int, warmup: int) -> dict:
    """Time decode steps of one (sequence, layer) slice -- every KV head of the
    model at full context -- through the reference's public API
    (KittyCacheState.insert_token + attend, cache.py:107-252) and extrapolate to
    the whole step (x global batch x layers)."""
    import numpy as np

    kv = _reference_module()
    kind = "reference" if kv is not None else "port"
    h_kv, h_q, ctx, frac = wl["h_kv"], wl["h_q"], wl["context"], wl["boost_fraction"]
    rng = np.random.default_rng(7)
    d = 128
    if kv is not None:
        st = kv.KittyCacheState(kv.KittyConfig(h_kv=h_kv, h_q=h_q, boost_fraction=frac))
    else:
        from oracle import kitty_oracle as ko

        st = ko.OracleCache(32, 128, 128, d, h_kv, h_q, frac)
    outl = rng.choice(d, OUTLIERS, replace=False)
    k = rng.standard_normal((h_kv, ctx, d)).astype(np.float32)
    k[..., outl] *= 8
    v = rng.standard_normal((h_kv, ctx, d)).astype(np.float32)
    t_setup = time.time()
    st.prefill(k, v)  # the reference's prefill: the fold of insert_token (cache.py:125-142)
    setup_s = time.time() - t_setup
    times = []
    for i in range(warmup + max(1, n_steps)):
        kn = rng.standard_normal((h_kv, d)).astype(np.float32)
        kn[:, outl] *= 8
        vn = rng.standard_normal((h_kv, d)).astype(np.float32)
        q = rng.standard_normal((h_q, d)).astype(np.float32)
        t0 = time.perf_counter()
        st.insert_token(kn, vn)
        st.attend(q)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    t_slice = sum(times) / len(times)
    step_s = t_slice * wl["global_batch"] * wl["layers"]
    return {
        "value": round(wl["global_batch"] / step_s, 4), "unit": "tokens/s", "step_s": step_s,
        "cores": len(os.sched_getaffinity(0)), "kind": kind, "cpu_model": _cpu_model(), "extrapolated": True,
        "sample": f"1 sequence x 1 layer x {h_kv} kv heads at {ctx} tokens per step (insert_token + attend, "
                  f"{t_slice * 1e3:.1f} ms, {'kittykv ' + getattr(kv, '__version__', '') if kv else 'oracle port'}), "
                  f"extrapolated x{wl['global_batch']} sequences x{wl['layers']} layers; setup (prefill fold) "
                  f"{setup_s:.1f} s untimed",
        "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default(all cores)"),
    }


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    wl = workload(args, world)
    cb = cpu_reference(wl, n_steps=args.steps, warmup=args.warmup)
    line = {
        "metric": METRIC,
        "impl": "reference",
        "value": cb["value"],
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(cb["step_s"] * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong" if wl["shard"] == "kv_head" else "weak",
        "vs_baseline": None,
        "dtype": "f32 (numpy)",
        "data": "synthetic: K ~ N(0,1) with 16 outlier channels x8, V,q ~ N(0,1)",
        "config": wl,
        "extrapolated": True,
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "extrapolated")},
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["kitty", "reference"], default="kitty")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--shard", choices=["request", "kv_head"], default=None,
                    help="multi-GPU partition (default: the config's: request for C1-C4, kv_head for C5)")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--context", type=int, default=0)
    ap.add_argument("--boost", type=float, default=None)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend for N > 1 (gloo: ranks may share one GPU, smoke tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this command under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_kitty(args)


if __name__ == "__main__":
    main()
