#!/usr/bin/env python3
"""Decode-attention benchmark of the Kitty hot path on B200.

Workload (BASELINE.json configs[1], fits one GPU): LLaMA3-8B attention shape
-- 32 layers, GQA 32 q / 8 kv heads, head_dim 128 -- batch 16, 32K context,
Kitty 2-bit K/V + 12.5 % boosted key channels.  One step = for every layer:
append one token (insert + pack when a q-buffer fills) and attend over the
whole cache with pages dequantised on the fly.  Metric: decode tokens/s
(= sequences / step time) and achieved HBM GB/s of the attention kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kitty|reference]

N > 1 runs under torchrun, one process per GPU; requests are partitioned
across ranks (weak scaling: each rank owns its own batch of 16) with no
collective on the data path.  The reference arm (--impl reference) times the
CPU oracle port of the reference (oracle/kitty_oracle.py, a restatement of
kittykv's numpy implementation) on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (layers, batch per GPU, context, h_kv, h_q, boost_fraction, description)
    "c1": (1, 1, 4096, 8, 32, 0.125, "single-layer synthetic: batch 1, 8 kv / 32 q heads, d 128, 4K context"),
    "c2": (32, 16, 32768, 8, 32, 0.125, "LLaMA3-8B attention shape (32 layers, GQA 32q/8kv, d=128), batch 16, 32K context"),
    "c3": (36, 64, 8192, 8, 32, 0.125, "Qwen3-8B attention shape (36 layers, GQA 32q/8kv, d=128), batch 64, 8K context"),
    "c4": (32, 1, 131072, 8, 32, 0.125, "LLaMA3-8B long context 128K, 1 request per GPU"),
    "c5": (80, 128, 16384, 8, 64, 0.125, "LLaMA3-70B attention shape (80 layers, GQA 64q/8kv), 16K context, batch 128 per GPU"),
}

OUTLIERS = 16  # outlier key channels (x8), SyntheticSpec-style (tensor_io.py:89-124)


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
# Kitty (GPU) arm
# ---------------------------------------------------------------------------


def run_kitty(args):
    import torch
    import torch.distributed as dist

    import paper_2511_18643_b200 as kb
    from paper_2511_18643_b200.decode import DecodeStep

    rank, world, local = _env_rank()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", torch.cuda.current_device())
    layers, batch, ctx, h_kv, h_q, frac, desc = CONFIGS[args.config]
    if args.layers:
        layers = args.layers
    if args.batch:
        batch = args.batch
    if args.context:
        ctx = args.context
    if args.boost is not None:
        frac = args.boost
    cfg = kb.KittyConfig(h_kv=h_kv, h_q=h_q, boost_fraction=frac)
    steps, warmup = args.steps, args.warmup
    max_tokens = ctx + warmup + steps + 2 * (warmup + steps) + 8
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    step = DecodeStep(cfg, layers, batch, max_tokens, dev)

    # -- synthetic prefill (not timed): K ~ N(0,1) with x8 outlier channels, V ~ N(0,1), bf16
    outl = torch.randperm(cfg.d, generator=gen, device=dev)[:OUTLIERS]
    gain = torch.ones(cfg.d, device=dev)
    gain[outl] = 8.0
    t0 = time.time()
    chunk = max(1, min(batch, (1 << 31) // (cfg.h_kv * ctx * cfg.d * 2)))
    for cache in step.layers:
        for b0 in range(0, batch, chunk):
            nb = min(chunk, batch - b0)
            k = (torch.randn((nb, cfg.h_kv, ctx, cfg.d), generator=gen, device=dev) * gain).bfloat16()
            v = torch.randn((nb, cfg.h_kv, ctx, cfg.d), generator=gen, device=dev).bfloat16()
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

    def one(i):
        step.k_in.copy_(ks[i])
        step.v_in.copy_(vs[i])
        step.q_in.copy_(qs[i])
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
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop()
    ms_per_step = ms / steps
    for c in step.layers:
        c.check()

    # -- attention kernel alone (attention + split-KV combine of every layer), captured
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

    # -- e2e: host (pinned) inputs -> device, step, outputs -> host, per step.
    # Copies are pipelined as a serving loop would: step i + 1's inputs go
    # host -> device staging on a copy stream while step i computes, step i's
    # outputs are staged on the device and read back during step i + 1; every
    # step's copies stay inside the timed region (the last read-back included).
    host_k = ks[warmup:].cpu().pin_memory()
    host_v = vs[warmup:].cpu().pin_memory()
    host_q = qs[warmup:].cpu().pin_memory()
    e_steps = steps  # every timed step (the pipeline fill / drain amortised as in the device timing)
    host_out = [torch.empty(step.out.shape, dtype=step.out.dtype).pin_memory() for _ in range(e_steps)]
    st_in = [(torch.empty_like(step.k_in), torch.empty_like(step.v_in), torch.empty_like(step.q_in)) for _ in range(2)]
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
            for dst, src in zip(st_in[i % 2], (host_k[i], host_v[i], host_q[i])):
                dst.copy_(src, non_blocking=True)
            in_ready[i % 2].record(cp)

    if not pipelined:
        for i in range(e_steps):
            step.k_in.copy_(host_k[i], non_blocking=True)
            step.v_in.copy_(host_v[i], non_blocking=True)
            step.q_in.copy_(host_q[i], non_blocking=True)
            step.step()
            host_out[i].copy_(step.out, non_blocking=True)
    h2d(0) if pipelined else None
    for i in range(e_steps if pipelined else 0):
        if i + 1 < e_steps:
            h2d(i + 1)
        main.wait_event(in_ready[i % 2])
        step.k_in.copy_(st_in[i % 2][0])
        step.v_in.copy_(st_in[i % 2][1])
        step.q_in.copy_(st_in[i % 2][2])
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
    e_ms = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    assert all(torch.isfinite(h.float()).all() for h in host_out)
    e2e_tps = batch * world / (e_ms / e_steps * 1e-3)

    bytes_step = layers * bytes_per_launch
    tps = batch * world / (ms_per_step * 1e-3)
    traffic = _ncu_traffic(args.config)
    launches = steps * step.launches_per_step()
    line = {
        "metric": "decode-attn tokens/sec and achieved HBM GB/s (% of roofline) at 1/2/4/8 B200",
        "value": round(tps, 2),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 2-bit codes -> fp16 MMA / fp32 accumulate (bf16 in/out)",
        "data": "synthetic: K ~ N(0,1) with 16 outlier channels x8, V,q ~ N(0,1), rounded to bf16; random-init, no checkpoint",
        "config": {
            "workload": desc, "config": args.config, "layers": layers, "global_batch": batch * world,
            "batch_per_gpu": batch, "context": ctx, "h_kv": h_kv, "h_q": h_q, "head_dim": cfg.d,
            "boost_fraction": frac, "d_boost": cfg.d_boost, "parallelism": f"request-sharded x{world}",
            "cuda_graph": use_graph,
            "l2": f"working set {bytes_step / 1e9:.2f} GB/step >> 126 MB L2 (no flush needed)",
            "prefill_s": round(prefill_s, 2),
        },
        "hbm_gbs_step": round(bytes_step / (ms_per_step * 1e-3) / 1e9, 1),
        "roofline": {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "peak_kind": peak_kind, "kernel": "kitty decode attention (per layer launch)",
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(attn_avg_ms, 4),
            "launch_timing": f"graph of {layers} attention+combine launches x {reps} replays, CUDA events",
            "frac_of_8TBs": round(achieved / 8000.0, 4),
        },
        "e2e": {
            "value": round(e2e_tps, 2), "unit": "tokens/s",
            "h2d_bytes_per_step": step.input_bytes(), "d2h_bytes_per_step": step.output_bytes(),
            "steps": e_steps,
            "copies": ("pinned host <-> device every step, pipelined on a copy stream (step i+1 H2D and step i D2H overlap compute)"
                       if pipelined else "pinned host <-> device every step, on the compute stream"),
        },
        "gpu_launches": launches,
        "clocks": clk,
        "wall_s_timed": round(wall, 3),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, layers, batch, ctx, h_kv, h_q, frac, n_steps=1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _ncu_traffic(config):
    """DRAM bytes per attention launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of kittykv, numpy / OpenBLAS on host cores)
# ---------------------------------------------------------------------------


def _cpu_slice_setup(ctx, h_kv, h_q, frac, seed=7):
    import numpy as np

    from oracle import kitty_oracle as ko

    rng = np.random.default_rng(seed)
    d = 128
    st = ko.OracleCache(32, 128, 128, d, h_kv, h_q, frac)
    outl = rng.choice(d, OUTLIERS, replace=False)
    # the reference's prefill is the fold of insert_token (cache.py:125-142)
    k = rng.standard_normal((h_kv, ctx, d)).astype(np.float32)
    k[..., outl] *= 8
    v = rng.standard_normal((h_kv, ctx, d)).astype(np.float32)
    st.prefill(k, v)
    return st, rng, outl


def cpu_baseline(args, layers, batch, ctx, h_kv, h_q, frac, n_steps=1):
    """Time the oracle port on one (sequence, layer) slice -- all KV heads at
    full context -- and extrapolate to the whole step (x batch x layers)."""
    import numpy as np

    cores = len(os.sched_getaffinity(0))
    t_setup = time.time()
    st, rng, outl = _cpu_slice_setup(ctx, h_kv, h_q, frac)
    setup_s = time.time() - t_setup
    times = []
    for _ in range(max(1, n_steps)):
        k = rng.standard_normal((h_kv, 128)).astype(np.float32)
        k[:, outl] *= 8
        v = rng.standard_normal((h_kv, 128)).astype(np.float32)
        q = rng.standard_normal((h_q, 128)).astype(np.float32)
        t0 = time.perf_counter()
        st.insert_token(k, v)
        st.attend(q)
        times.append(time.perf_counter() - t0)
    t_slice = min(times)
    step_s = t_slice * batch * layers
    return {
        "value": round(batch / step_s, 4),
        "unit": "tokens/s",
        "cores": cores,
        "kind": "port",
        "sample": f"1 sequence x 1 layer x {h_kv} kv heads at {ctx} tokens (insert_token + attend, "
                  f"{t_slice * 1e3:.1f} ms), extrapolated x{batch} sequences x{layers} layers; "
                  f"setup (prefill fold) {setup_s:.1f} s untimed",
        "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default(all cores)"),
    }


def run_reference(args):
    rank, world, _ = _env_rank()
    layers, batch, ctx, h_kv, h_q, frac, desc = CONFIGS[args.config]
    if args.layers:
        layers = args.layers
    if args.batch:
        batch = args.batch
    if args.context:
        ctx = args.context
    if args.boost is not None:
        frac = args.boost
    if rank != 0:
        return
    import numpy as np

    cores = len(os.sched_getaffinity(0))
    st, rng, outl = _cpu_slice_setup(ctx, h_kv, h_q, frac)
    times = []
    for i in range(args.warmup + args.steps):
        k = rng.standard_normal((h_kv, 128)).astype(np.float32)
        k[:, outl] *= 8
        v = rng.standard_normal((h_kv, 128)).astype(np.float32)
        q = rng.standard_normal((h_q, 128)).astype(np.float32)
        t0 = time.perf_counter()
        st.insert_token(k, v)
        st.attend(q)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    t_slice = sum(times) / len(times)
    step_s = t_slice * batch * layers
    value = batch / step_s
    line = {
        "metric": "decode-attn tokens/sec and achieved HBM GB/s (% of roofline) at 1/2/4/8 B200",
        "impl": "reference",
        "value": round(value, 4),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_s * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (numpy)",
        "data": "synthetic: K ~ N(0,1) with 16 outlier channels x8, V,q ~ N(0,1)",
        "config": {"workload": desc, "config": args.config, "layers": layers, "global_batch": batch,
                   "context": ctx, "h_kv": h_kv, "h_q": h_q, "boost_fraction": frac},
        "cpu_baseline": {
            "value": round(value, 4), "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": f"each step: 1 sequence x 1 layer x {h_kv} kv heads at {ctx} tokens "
                      f"(insert_token + attend, {t_slice * 1e3:.1f} ms), extrapolated x{batch} x{layers}",
        },
        "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["kitty", "reference"], default="kitty")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--context", type=int, default=0)
    ap.add_argument("--boost", type=float, default=None)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_kitty(args)


if __name__ == "__main__":
    main()
