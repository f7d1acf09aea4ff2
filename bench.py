#!/usr/bin/env python
"""RDKV decode benchmark on B200 (BASELINE.json metric: decode tok/s & us/step at
128K context; HBM GB/s vs peak; speedup vs FP16 full-KV).

Workload (BASELINE.json configs[2] at N=1): LLaMA-3.1-8B KV shape (32 layers,
32 q / 8 kv heads, d=128), 128K context, 128 FP16-equivalent tokens per layer,
16 sequences per GPU (weak scaling). Prefill-time allocate+pack runs once in
setup; one timed *step* = packed decode attention of one new token for every
(sequence, layer, KV head) tile and all 4 GQA query heads (one launch).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun each rank packs and decodes its own 16 sequences (no data-path
collective); the step time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--batch", type=int, default=16, help="sequences per GPU")
    p.add_argument("--layers", type=int, default=32)
    p.add_argument("--ctx", type=int, default=131072)
    p.add_argument("--n-tokens", type=int, default=128)
    p.add_argument("--zc", type=int, default=0, help="Zone C tokens appended per tile before timing")
    p.add_argument("--hh", action="store_true", help="heavy-hitter synthetic cache (mixed bit tiers)")
    p.add_argument("--kernel", type=int, default=0, help="0 auto, 1 generic, 2 tensor-core")
    p.add_argument("--no-fp16-baseline", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-pipeline", action="store_true")
    p.add_argument("--no-secondary", action="store_true", help="skip the Zone C / budget-512 secondary lines")
    p.add_argument("--cpu-budget-s", type=float, default=8.0)
    p.add_argument("--shard", default="seqs", choices=["seqs", "heads"],
                   help="multi-GPU partition: seqs = batch sequences per GPU (weak scaling); "
                        "heads = the batch on every GPU, KV heads split across GPUs (strong scaling)")
    p.add_argument("--dist-backend", default=None, choices=["nccl", "gloo"],
                   help="process-group backend (default nccl; gloo lets several ranks share one GPU)")
    return p.parse_args()


# ---------------------------------------------------------------------------------
def check_env():
    """The product library reads no environment knobs; a debug build's timing
    knobs (RDKV_DECODE_NULL etc., csrc/Makefile EXPERIMENTS=1) must not be set
    for a bench run, whatever library is loaded."""
    bad = sorted(k for k in os.environ if k.startswith("RDKV_DECODE_"))
    if bad:
        raise SystemExit(f"bench.py: unset the decode experiment knobs {bad} before timing")


def host_cpu():
    """CPU model and usable core count of the box."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count()
    return {"cpu_model": model, "nproc": n}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clocks / throttle reasons while the timed loop runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
               0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append(mhz)
                self.reasons |= int(r) & ~0x1
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def report(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def dist_setup(backend=None):
    from paper_2605_08317_b200 import dist as D

    return D.init(backend)


def barrier_sync(world):
    from paper_2605_08317_b200 import dist as D

    D.barrier_sync(world)


def max_over_ranks(x, world):
    from paper_2605_08317_b200 import dist as D

    return D.max_over_ranks(x, world)


# ---------------------------------------------------------------------------------
def reference_sample(spec, cfg_kwargs, budget_s):
    """The reference CPU path on one (sequence 0, layer 0) slice of the same synthetic
    workload: allocate_model + build_packed_model (oracle/_ref = the unmodified
    reference core), then packed_decode_step for all 32 q-heads through the
    reference's parallel_for, repeated for ~budget_s. Returns timing + outputs."""
    import oracle
    from paper_2605_08317_b200.workload import chunk_seed

    orc = oracle.load()
    ref = oracle.load_ref() if oracle.ref_available() else None
    lib = ref if ref is not None else orc
    H, T, d, g, Sw = spec.kv_heads, spec.ctx, spec.head_dim, spec.group, spec.probe_rows
    # enough (sequence 0, layer) slices that the reference's parallel_for over
    # (layer, kv-head) items has at least one item per host core
    ncores = os.cpu_count() or 1
    Ls = max(1, min(spec.layers, -(-ncores // H))) if ref is not None else 1
    ks, vs, pqs = [], [], []
    for layer in range(Ls):
        s = chunk_seed(spec.seed, spec.first_seq, layer)
        ks.append(orc.gen_counter(s, 0, 0, H * T * d, d, T, spec.outlier_channels, spec.outlier_scale,
                                  spec.hh_stride, spec.hh_boost).reshape(H, T, d))
        vs.append(orc.gen_counter(s, 1, 0, H * T * d, d, T).reshape(H, T, d))
        pqs.append(orc.gen_counter(s, 2, 0, H * g * Sw * d, d, T, 0, 1.0, spec.hh_stride).reshape(H * g, Sw, d))
    k, v, pq = np.stack(ks), np.stack(vs), np.stack(pqs)
    q = np.stack([orc.gen_counter(QSEED + layer, 2, 0, H * g * d, d, T).reshape(H * g, d) for layer in range(Ls)])
    cfg = oracle.default_config(**cfg_kwargs)
    t0 = time.perf_counter()
    info = {"kind": "reference" if ref is not None else "port", "slices": Ls}
    if ref is not None:
        model = oracle.RefModel(ref, k, v, pq, cfg)
        info["alloc_s"], info["pack_s"] = model.alloc_seconds, model.pack_seconds
        heads = [model.head(0, h) for h in range(H)]
        out, _ = model.decode(q)
        times = []
        t_end = time.perf_counter() + budget_s
        while time.perf_counter() < t_end or len(times) < 3:
            _, sec = model.decode(q)
            times.append(sec)
        cores = ref.lib.ref_worker_count()
    else:  # port: serial oracle
        heads, tzs = [], []
        for h in range(H):
            r = orc.allocate_head(k[0, h], pq[0, h * g:(h + 1) * g], H, cfg)
            heads.append(r)
            tzs.append(orc.tz_build(k[0, h], v[0, h], r["v_bits"], r["k_bits"]))
        out = np.stack([tzs[j // g].decode(q[0, j]) for j in range(H * g)])[None]
        times = []
        t_end = time.perf_counter() + budget_s
        while time.perf_counter() < t_end or len(times) < 3:
            t1 = time.perf_counter()
            for j in range(H * g):
                tzs[j // g].decode(q[0, j])
            times.append(time.perf_counter() - t1)
        cores = 1
    info["setup_s"] = time.perf_counter() - t0
    info["sample_step_s"] = statistics.median(times) / Ls  # per (sequence, layer) slice
    info["cores"] = cores
    info["heads"] = heads
    info["out"] = out[:1]
    info["q"] = q[:1]
    return info


QSEED = 0xD15C0


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU path, rank 0 only."""
    if rank != 0:
        return
    from paper_2605_08317_b200.workload import WorkloadSpec

    spec = WorkloadSpec(batch=args.batch, layers=args.layers, ctx=args.ctx, n_tokens=args.n_tokens,
                        hh_stride=64 if args.hh else 0, hh_boost=1.0 if args.hh else 0.0)
    per_step = max(0.2, args.cpu_budget_s / max(args.steps, 1))
    info = reference_sample(spec, dict(n_tokens=spec.n_tokens, window=spec.probe_rows), per_step * args.steps)
    sample_units = spec.kv_heads  # one (sequence, layer) slice = 8 tiles, 32 q-heads
    seqs = spec.batch * (args.gpus if args.shard == "seqs" else 1)  # sequences in the whole job
    scale = (seqs * spec.layers * spec.kv_heads) / sample_units
    step_s = info["sample_step_s"] * scale
    value = seqs / step_s
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.shard == "seqs" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (K0 counter-based generator, FP16-representable)",
        "impl": "reference",
        "config": workload_config(spec, args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": info["cores"], "kind": info["kind"], **host_cpu(),
                         "sample": f"{info['slices']} of {int(scale)} (sequence, layer) slices (8 KV heads x 4 q-heads each, "
                                   f"T={spec.ctx}) decoded together through parallel_for: "
                                   f"{info['sample_step_s'] * 1e3:.3f} ms per slice; step = x{int(scale)}"},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "decode tok/s & us/step at 128K ctx; HBM GB/s vs peak; speedup vs FP16 full-KV"


def workload_config(spec, args, world):
    seqs = spec.batch * (world if args.shard == "seqs" else 1)
    part = (f"shard by sequence x{world} (weak scaling, no collective)" if args.shard == "seqs" else
            f"shard by KV head x{world} (strong scaling: every GPU holds the {spec.batch} sequences and "
            f"{spec.kv_heads // world}-{-(-spec.kv_heads // world)} of the {spec.kv_heads} KV heads; no collective)")
    return {
        "workload": f"LLaMA-3.1-8B KV shape ({spec.layers} layers, {spec.q_heads} q / {spec.kv_heads} kv heads, "
                    f"d={spec.head_dim}), {spec.ctx} ctx, {spec.n_tokens}-token/layer budget, batch {spec.batch}/GPU, "
                    "one decode step over all layers (configs[2])",
        "layers": spec.layers, "q_heads": spec.q_heads, "kv_heads": spec.kv_heads, "head_dim": spec.head_dim,
        "ctx": spec.ctx, "batch_per_gpu": spec.batch if args.shard == "seqs" else f"{spec.batch} (KV-head shard)",
        "global_batch": seqs, "n_tokens": spec.n_tokens, "zone_c": args.zc, "heavy_hitters": bool(args.hh),
        "parallelism": part, "shard": args.shard,
        "l2": "inputs larger than L2: step i decodes rotation copy i % NR of the packed arena, q and out "
              "(NR copies >= 3x the 126 MB L2), K steps back to back from one CUDA graph",
        "io": "fp16 q/out",
    }


# ---------------------------------------------------------------------------------
def fp16_fullkv_baseline(spec, steps, warmup):
    """FlashInfer 0.6.11 batch decode over an FP16 paged full KV cache (same shapes).
    One layer's KV (batch x 128K) is resident; a step runs it for all layers."""
    import torch

    # prebuilt (cross-compiled) FlashInfer module, see baseline/prebuild_flashinfer.py
    os.environ.setdefault("FLASHINFER_WORKSPACE_BASE", os.path.join(ROOT, "baseline", "flashinfer_ws"))
    os.environ.setdefault("FLASHINFER_CUDA_ARCH_LIST", "10.0a")
    import flashinfer

    B, T, H, Hq, d = spec.batch, spec.ctx, spec.kv_heads, spec.q_heads, spec.head_dim
    page = 16
    pps = T // page
    kv = torch.empty((B * pps, 2, page, H, d), dtype=torch.float16, device="cuda").normal_()
    indptr = (torch.arange(B + 1, dtype=torch.int32, device="cuda") * pps)
    indices = torch.arange(B * pps, dtype=torch.int32, device="cuda")
    last = torch.full((B,), page, dtype=torch.int32, device="cuda")
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=True)
    w.plan(indptr, indices, last, Hq, H, d, page, q_data_type=torch.float16, kv_data_type=torch.float16)
    q = torch.randn((B, Hq, d), dtype=torch.float16, device="cuda")
    out = torch.empty_like(q)
    for _ in range(max(warmup, 2)):
        w.run(q, kv, out=out)
    torch.cuda.synchronize()
    n = max(2, min(steps, 10))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(n):
        for _layer in range(spec.layers):
            w.run(q, kv, out=out)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / n
    bytes_step = spec.layers * (B * T * H * d * 2 * 2 + 2 * B * Hq * d * 2)
    del kv
    torch.cuda.empty_cache()
    return {"impl": f"flashinfer {flashinfer.__version__} BatchDecodeWithPagedKVCacheWrapper (fp16, tensor cores, page 16)",
            "ms_per_step": ms, "tok_s": B / (ms / 1e3), "GB_s": bytes_step / (ms / 1e3) / 1e9,
            "bytes_per_step": bytes_step}


def pipeline_config2(P, steps):
    """configs[1]: 32 layers, 32K context, batch 1 — full allocate+pack+decode on 1 B200."""
    import torch
    from paper_2605_08317_b200.workload import WorkloadSpec, build

    spec = WorkloadSpec(batch=1, layers=32, ctx=32768, n_tokens=128, seed=2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model, timing, _, _ = build(spec)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    q = P.generate((model.units, spec.group, spec.head_dim), torch.float16, seed=QSEED, tensor=2)
    out = torch.empty_like(q)
    for _ in range(5):
        P.packed_decode_step(model, q, out)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(steps):
        P.packed_decode_step(model, q, out)
    e[1].record()
    torch.cuda.synchronize()
    return {"config": "configs[1]: LLaMA-3.1-8B shape, 32 layers, 32K ctx, batch 1 (allocate+pack+decode)",
            "allocate_pack_s": setup, **{k: round(v, 4) for k, v in timing.items()},
            "decode_us_per_step": e[0].elapsed_time(e[1]) / steps * 1e3,
            "note": "allocate/pack timed per (layer) chunk incl. host syncs; decode back-to-back (L2-warm)"}


def graph_step_us(P, model, q, steps, kernel=0, split=1):
    """Back-to-back decode steps from one CUDA graph over rotation copies of the
    arena (>= 3x L2), one event pair: the same method as the headline number."""
    import torch

    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    per_copy = model.arena_bytes + 2 * q.numel() * q.element_size()
    n_rot = max(1, -(-3 * l2 // per_copy))
    rot = []
    for r in range(n_rot):
        m = P.PackedModel(model.arena if r == 0 else model.arena.clone(), model.offsets, model.offsets_host,
                          model.units, model.group, model.head_dim, model.zc_k, model.zc_v, model.zc_len, model.zc_cap,
                          model.zc_count)
        m.share_plan(model)
        rot.append((m, q if r == 0 else q.clone(), torch.empty_like(q)))
    for i in range(3):
        m, qq, oo = rot[i % n_rot]
        P.packed_decode_step(m, qq, oo, kernel=kernel, split=split, workspace=m.split_ws if split > 1 else None)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=side):
        for i in range(steps):
            m, qq, oo = rot[i % n_rot]
            P.packed_decode_step(m, qq, oo, kernel=kernel, split=split,
                                 workspace=m.split_ws if split > 1 else None)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        e0.record(side)
        g.replay()
        e1.record(side)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3, n_rot


def secondary_configs(P, spec0, model, q, args):
    """Other BASELINE shapes on the same GPU (secondary lines, not the headline):
    the decode step with the new token already appended to Zone C, and a
    configs[3]-style budget point (512 FP16-equivalent tokens per layer)."""
    import torch
    from paper_2605_08317_b200.workload import WorkloadSpec, build

    out = {}
    U, d = model.units, spec0.head_dim
    peak, _ = load_peaks()
    # (1) Zone C: the step's own token appended (append_new_token, trizone.cpp:307-314)
    model.zc_cap, model.zc_count = 16, 0
    model.zc_k = torch.zeros((U, 16, d), dtype=torch.float16, device="cuda")
    model.zc_v = torch.zeros_like(model.zc_k)
    model.zc_len = torch.zeros(U, dtype=torch.int32, device="cuda")
    kn = P.generate((U, d), torch.float16, seed=77, tensor=1)
    P.append_new_token(model, kn, kn)
    us, _ = graph_step_us(P, model, q, min(args.steps, 100))
    byts = model.survey_bytes(io_bytes=2)
    out["zone_c_1"] = {"config": "configs[2] step with the new token in Zone C (1 fp16 K/V row per tile)",
                       "us_per_step": us, "tok_s": spec0.batch / (us / 1e6),
                       "roofline_frac": byts / (us / 1e6) / 1e9 / peak}
    # (2) a generation loop on the device: per step append the new token's K/V
    # to Zone C (rdkv_cuda_append) and decode, 16 steps replayed from one CUDA
    # graph (Zone C reset at the start of each replay)
    nsteps = 16
    model.zc_cap, model.zc_count = nsteps, 0
    model.zc_k = torch.zeros((U, nsteps, d), dtype=torch.float16, device="cuda")
    model.zc_v = torch.zeros_like(model.zc_k)
    model.zc_len = torch.zeros(U, dtype=torch.int32, device="cuda")
    kv = [P.generate((U, d), torch.float16, seed=900 + i, tensor=1) for i in range(nsteps)]
    qs = [P.generate(tuple(q.shape), torch.float16, seed=700 + i, tensor=2) for i in range(nsteps)]
    o = torch.empty_like(q)
    # token step i decodes rotation copy i % n of the packed arena (>= 3x L2 in total), all
    # copies sharing the one Zone C that the loop appends to: the packed tiles stream from HBM
    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    n_rot = max(2, -(-3 * l2 // model.arena_bytes))
    views = [model]
    for r in range(1, n_rot):
        mr = P.PackedModel(model.arena.clone(), model.offsets, model.offsets_host, U, model.group, d,
                           model.zc_k, model.zc_v, model.zc_len, model.zc_cap, 0)
        mr.share_plan(model)
        views.append(mr)

    def loop():
        model.zc_len.zero_()
        for mv in views:
            mv.zc_count = 0  # host mirror of the reset (append_new_token checks capacity)
        for i in range(nsteps):
            P.append_new_token(model, kv[i], kv[i])
            mv = views[i % n_rot]
            mv.zc_count = model.zc_count
            P.packed_decode_step(mv, qs[i], o)

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        loop()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        loop()
    g.replay()
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        e0.record(side)
        for _ in range(reps):
            g.replay()
        e1.record(side)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (reps * nsteps) * 1e3
    byts_loop = model.survey_bytes(io_bytes=2) + U * (nsteps + 1) / 2 * d * 2 * 2  # mean Zone C rows per step
    step_ms = getattr(args, "_step_ms", None)  # the headline (no Zone C) step of this run
    out["decode_loop_16"] = {"config": "16 generated tokens: append (Zone C) + decode per step, one CUDA graph; "
                                       f"Zone C grows 1..16 rows per tile; step i reads rotation copy i % {n_rot} "
                                       "of the arena (L2 cold for the packed tiles)",
                             "us_per_token_step": us, "tok_s": spec0.batch / (us / 1e6),
                             "vs_no_zone_c_step": us / (step_ms * 1e3) if step_ms else None,
                             "roofline_frac": byts_loop / (us / 1e6) / 1e9 / peak}
    del views
    model.zc_cap, model.zc_k, model.zc_v, model.zc_len = 0, None, None, None
    # (3) batch sweep (configs[2] is "batch 1-16"): the first b sequences of the
    # packed arena (a prefix of the units), same timing method
    sweep = {}
    for b in (1, 2, 4, 8):
        ub = b * spec0.layers * spec0.kv_heads
        sub = P.PackedModel(model.arena, model.offsets[: ub + 1], model.offsets_host[: ub + 1], ub, model.group,
                            model.head_dim)
        sub.prepare()
        us, _ = graph_step_us(P, sub, q[:ub].contiguous(), min(args.steps, 100))
        sweep[str(b)] = {"us_per_step": us, "tok_s": b / (us / 1e6)}
    out["batch_sweep"] = sweep
    # (4) configs[4]: LLaMA-3.1-70B shape (80 layers, 64 q / 8 kv heads: GQA group 8),
    # 128K ctx; batch 8 over 8 GPUs = one sequence per GPU
    spec70 = WorkloadSpec(batch=1, layers=80, q_heads=64, kv_heads=8, ctx=spec0.ctx, n_tokens=128, seed=5)
    m70, _, _, _ = build(spec70)
    q70 = P.generate((m70.units, spec70.group, d), torch.float16, seed=QSEED, tensor=2)
    us, _ = graph_step_us(P, m70, q70, min(args.steps, 100))
    byts = m70.survey_bytes(io_bytes=2)
    out["llama70b_1seq_per_gpu"] = {"config": "configs[4]: LLaMA-3.1-70B KV shape (80 layers, 64 q / 8 kv heads), "
                                              "128K ctx, n=128, one sequence per GPU (batch 8 over 8 GPUs)",
                                    "us_per_step": us, "tok_s_per_gpu": 1 / (us / 1e6),
                                    "roofline_frac": byts / (us / 1e6) / 1e9 / peak}
    del m70, q70
    # (5) heavy-hitter caches (the realistic attention shape: a few 4-bit rows / channels
    # in ~16% of the tiles): configs[2] shape with heavy-hitter injection
    spec_hh = WorkloadSpec(batch=spec0.batch, layers=spec0.layers, ctx=spec0.ctx, n_tokens=128, seed=1,
                           hh_stride=64, hh_boost=1.0)
    mhh, _, sthh, _ = build(spec_hh)
    qhh = P.generate((mhh.units, spec_hh.group, d), torch.float16, seed=QSEED, tensor=2)
    us, _ = graph_step_us(P, mhh, qhh, min(args.steps, 100))
    byts = mhh.survey_bytes(io_bytes=2)
    out["heavy_hitters"] = {"config": "configs[2] shape with heavy-hitter injection (every 64th key boosted): "
                                      "mixed 2/4-bit tiles", "us_per_step": us, "tok_s": spec_hh.batch / (us / 1e6),
                            "roofline_frac": byts / (us / 1e6) / 1e9 / peak,
                            "plan_uniform2": int(mhh.plan.uniform2),
                            "v4_rows": int(sum(s["n_kept"].sum() for s in sthh))}
    del mhh, qhh
    # (6) budget sweep point: 512 FP16-equivalent tokens per layer (~512 kept tokens per head)
    spec = WorkloadSpec(batch=spec0.batch, layers=spec0.layers, ctx=spec0.ctx, n_tokens=512, seed=3)
    m2, _, st2, _ = build(spec)
    q2 = P.generate((m2.units, spec.group, d), torch.float16, seed=QSEED, tensor=2)
    us, _ = graph_step_us(P, m2, q2, min(args.steps, 100))
    byts = m2.survey_bytes(io_bytes=2)
    out["budget_512"] = {"config": "LLaMA-3.1-8B KV shape, 128K ctx, n=512 tokens/layer (configs[3] budget point), "
                                   f"batch {spec.batch}, kept tokens/head {float(np.mean([s['n_kept'].mean() for s in st2])):.1f}",
                         "us_per_step": us, "tok_s": spec.batch / (us / 1e6),
                         "roofline_frac": byts / (us / 1e6) / 1e9 / peak, "bytes_per_step": byts}
    del m2, q2
    # (7) configs[3]: Mistral-7B / Qwen2.5-7B GQA shapes at 64K, budget sweep, with heavy hitters
    # and 4 outlier K channels (x8) so the V and K tiers span 2/4/8 bits
    c4 = {}
    for model, (L, Hq, Hkv), budgets in (("qwen2.5-7b", (28, 28, 4), (64, 256, 1024, 2048)),
                                         ("mistral-7b", (32, 32, 8), (64, 2048))):
        for n in budgets:
            spec = WorkloadSpec(batch=4, layers=L, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                                hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
            m4, _, st4, _ = build(spec)
            q4 = P.generate((m4.units, spec.group, d), torch.float16, seed=QSEED, tensor=2)
            us, _ = graph_step_us(P, m4, q4, min(args.steps, 50))
            byts = m4.survey_bytes(io_bytes=2)
            c4[f"{model}_n{n}"] = {"us_per_step": us, "tok_s": spec.batch / (us / 1e6),
                                   "roofline_frac": byts / (us / 1e6) / 1e9 / peak, "bytes_per_step": byts,
                                   "plan_uniform2": int(m4.plan.uniform2),
                                   "kept_per_head": float(np.mean([s["n_kept"].mean() for s in st4]))}
            del m4, q4
    out["configs3_gqa_64k_budget_sweep"] = {"config": "configs[3]: Qwen2.5-7B (28 layers, 28 q / 4 kv, g=7) and "
                                                      "Mistral-7B (32 layers, 32 q / 8 kv) KV shapes, 64K ctx, batch 4, "
                                                      "heavy hitters + 4 outlier K channels x8", "points": c4}
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    check_env()
    world, rank, local = dist_setup(args.dist_backend)
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return
    import torch

    from paper_2605_08317_b200 import capi
    from paper_2605_08317_b200 import pipeline as P
    from paper_2605_08317_b200.workload import WorkloadSpec, build

    capi.lib()
    spec = WorkloadSpec(batch=args.batch, layers=args.layers, ctx=args.ctx, n_tokens=args.n_tokens, rank=rank,
                        hh_stride=64 if args.hh else 0, hh_boost=1.0 if args.hh else 0.0, zc_cap=max(args.zc, 0),
                        shard=args.shard, world=world)
    seqs_job = spec.batch * (world if args.shard == "seqs" else 1)  # sequences decoded per step, all ranks
    t0 = time.perf_counter()
    model, build_timing, stats, first_alloc = build(spec)
    build_s = time.perf_counter() - t0
    U, g, d = model.units, spec.group, spec.head_dim
    if args.zc:
        for _ in range(args.zc):
            kn = P.generate((U, d), torch.float16, seed=77, tensor=1)
            P.append_new_token(model, kn, kn)
    q = P.generate((U, g, d), torch.float16, seed=QSEED, tensor=2)
    out = torch.empty_like(q)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    # Inputs larger than L2 between timed steps: step i decodes rotation copy
    # i % NR of the packed arena (+ its own q / out), NR copies spanning >= 3x L2,
    # so every step streams its tiles from HBM. The K steps are launched back to
    # back from one CUDA graph (what a serving loop does) and timed with one
    # pair of device events.
    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    per_copy = model.arena_bytes + 2 * q.numel() * q.element_size()
    n_rot = max(2, -(-3 * l2 // per_copy))
    rot = [(model, q, out)]
    for r in range(1, n_rot):
        m = P.PackedModel(model.arena.clone(), model.offsets, model.offsets_host, U, g, d,
                          model.zc_k, model.zc_v, model.zc_len, model.zc_cap, model.zc_count)
        m.share_plan(model)
        rot.append((m, q.clone(), torch.empty_like(out)))

    def step(i):
        m, qq, oo = rot[i % n_rot]
        P.packed_decode_step(m, qq, oo, kernel=args.kernel)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=side):
        for i in range(args.steps):
            step(i)
    torch.cuda.synchronize()
    graph.replay()  # untimed: first replay uploads the graph
    torch.cuda.synchronize()
    # ---- timed region: K decode steps back to back, device events on the graph's stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    barrier_sync(world)
    with sampler:
        with torch.cuda.stream(side):
            ev0.record(side)
            graph.replay()
            ev1.record(side)
        barrier_sync(world)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local, world)
    value = seqs_job / (ms / 1e3)
    last = min(n_rot, args.steps) - 1  # the last rotation copy the timed steps decoded
    assert torch.equal(rot[0][2], rot[last][2])
    del graph

    # ---- the same step timed alone after an L2 flush (one event pair per step):
    # includes launch latency and a cold L2 every step
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    nf = min(args.steps, 50)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(nf)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(nf)]
    for i in range(nf):
        flush.zero_()
        starts[i].record(stream)
        step(0)
        ends[i].record(stream)
    torch.cuda.synchronize()
    flushed_ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / nf, world)

    # ---- end to end through the C-ABI with pinned host buffers: every step moves
    # its q from host memory to the GPU and its out back (rdkv_cuda_decode_host:
    # zero-copy, the kernel streams q in and out over PCIe with TMA bulk copies);
    # L2 flushed before each step
    import ctypes as C

    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    L = capi.lib()
    args_c = P.decode_args(model, q, out, 1, args.kernel)

    def e2e_run(call):
        st_ = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        en_ = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for _ in range(max(args.warmup, 3)):
            call()
        barrier_sync(world)
        for i in range(args.steps):
            flush.zero_()
            st_[i].record(stream)
            call()
            en_[i].record(stream)
        barrier_sync(world)
        return max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(st_, en_)) / args.steps, world)

    oh.zero_()
    e2e_ms = e2e_run(lambda: L.rdkv_cuda_decode_host(C.byref(args_c), qh.data_ptr(), oh.data_ptr(),
                                                     stream.cuda_stream))
    assert torch.equal(oh.cuda(), out)
    # the copy-engine variant (H2D / decode / D2H in 8 overlapped chunks), for reference
    dec = P.HostDecoder(model, q.dtype, chunks=8, kernel=args.kernel)
    oh.zero_()
    pipelined_ms = e2e_run(lambda: dec.step(qh, oh, stream.cuda_stream))
    assert torch.equal(oh.cuda(), out)
    dec.close()

    # ---- roofline of the decode kernel
    peak, peak_kind = load_peaks()
    # SURVEY.md §8(d) bytes (the allocation's own codes, params, map, q, out) are
    # the roofline's numerator; what the tile layout adds on top (header, 16-bit
    # perm entries, class padding) is reported beside it, not counted
    alg_bytes = model.survey_bytes(io_bytes=2)
    layout_bytes = model.decode_bytes(io_bytes=2)
    achieved = alg_bytes / (ms_local / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "decode_ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            if pj.get("units") == U and pj.get("kernel_mode") == args.kernel and pj.get("arena_bytes") == model.arena_bytes:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None

    # ---- per-layer launches (honest model-integrated number: one launch per layer)
    per_layer = None
    try:
        per_layer = per_layer_launch_ms(P, model, spec, q, out, flush, args)
    except Exception as e:  # noqa: BLE001
        per_layer = {"error": str(e)[:200]}

    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "us_per_step": ms * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.shard == "seqs" else "strong", "vs_baseline": None,
        "dtype": "fp32-accum/fp16-io, int codes",
        "data": "synthetic (K0 counter-based N(0,1)-like KV, FP16-representable), random-init",
        "config": workload_config(spec, args, world),
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "layout_bytes_per_launch": layout_bytes,
                     "layout_overhead_bytes": layout_bytes - alg_bytes,
                     "frac_incl_layout_overhead": layout_bytes / (ms_local / 1e3) / 1e9 / peak},
        "e2e": {"value": seqs_job / (e2e_ms / 1e3), "unit": "tok/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": qh.numel() * qh.element_size(),
                "d2h_bytes_per_step": oh.numel() * oh.element_size(),
                "path": "rdkv_cuda_decode_host (C-ABI), pinned host q/out: the kernel reads q over PCIe (TMA "
                        "bulk loads) and writes out (TMA bulk stores) inside the step",
                "copy_engine_pipelined_ms_per_step": pipelined_ms},
        "clocks": sampler.report(),
        "flushed_step": {"ms_per_step": flushed_ms, "tok_s": seqs_job / (flushed_ms / 1e3),
                         "note": "one launch per event pair after a 512 MiB memset (cold L2 + launch latency)"},
        "rotation_copies": n_rot,
        "per_layer_launch": per_layer,
        "setup": {"build_s": round(build_s, 2), **{k: round(v, 3) for k, v in build_timing.items()},
                  "arena_bytes": model.arena_bytes,
                  "kept_tokens_mean": float(np.mean([s["n_kept"].mean() for s in stats])),
                  "v16_rows": int(sum(s["n_v16"].sum() for s in stats))},
    }
    if rank == 0 and not args.no_fp16_baseline:
        try:
            fb = fp16_fullkv_baseline(spec, args.steps, args.warmup)
            fb["speedup_ours_vs_fp16"] = fb["ms_per_step"] / ms
            line["fp16_fullkv"] = fb
        except Exception as e:  # noqa: BLE001
            line["fp16_fullkv"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            info = reference_sample(spec, dict(n_tokens=spec.n_tokens, window=spec.probe_rows), args.cpu_budget_s)
            scale = spec.batch * spec.layers
            cpu_step = info["sample_step_s"] * scale
            line["cpu_baseline"] = {"value": spec.batch / cpu_step, "unit": "tok/s", "cores": info["cores"],
                                    "kind": info["kind"], **host_cpu(),
                                    "sample": f"sequence 0, layers 0..{info['slices'] - 1} (8 KV heads, 32 q-heads each, "
                                              f"T={spec.ctx}) decoded together through parallel_for: "
                                              f"{info['sample_step_s'] * 1e3:.3f} ms per slice x {scale} slices",
                                    "alloc_s_sample": info.get("alloc_s"), "pack_s_sample": info.get("pack_s")}
            # parity on the same slice: allocation and decode outputs vs the reference
            vb, kb, st = first_alloc
            match = all(np.array_equal(vb[h], info["heads"][h]["v_bits"]) and
                        np.array_equal(kb[h][: len(info["heads"][h]["k_bits"])], info["heads"][h]["k_bits"])
                        for h in range(spec.kv_heads))
            q0 = torch.from_numpy(info["q"][0].reshape(spec.kv_heads, g, d)).cuda().half()
            sub = P.PackedModel(model.arena, model.offsets, model.offsets_host, spec.kv_heads, g, d)
            sub.share_plan(model)
            sub.unit_ids = None  # a prefix of the units: no split lists
            o0 = P.packed_decode_step(sub, q0).float().cpu().numpy().reshape(-1, d)
            want = info["out"][0]
            err = float(max(np.linalg.norm(o0[j] - want[j]) / np.linalg.norm(want[j]) for j in range(len(want))))
            line["parity"] = {"slice": "sequence 0, layer 0 (8 KV heads, T=%d)" % spec.ctx,
                              "allocation_bit_exact": bool(match), "decode_max_rel_err": err,
                              "tolerance": 1e-3}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    if rank == 0 and world == 1 and not args.no_secondary:
        args._step_ms = ms
        try:
            line["secondary"] = secondary_configs(P, spec, model, q, args)
        except Exception as e:  # noqa: BLE001
            line["secondary"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if rank == 0 and world == 1 and not args.no_pipeline:
        try:
            pj = pipeline_config2(P, 50)
            print(json.dumps({"pipeline": pj}), file=sys.stderr, flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"pipeline_error": str(e)[:300]}), file=sys.stderr, flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def per_layer_launch_ms(P, model, spec, q, out, flush, args):
    """One launch per layer (what a model-integrated decode does), captured in a CUDA graph."""
    import torch

    subs = []
    H = spec.local_heads
    for layer in range(spec.layers):
        # units of this layer across the batch are not contiguous; build a per-layer offsets view
        idx = np.array([(b * spec.layers + layer) * H + h for b in range(spec.batch) for h in range(H)])
        offs = np.concatenate([model.offsets_host[idx], [0]])
        sub = P.PackedModel(model.arena, torch.from_numpy(offs).cuda(), offs, len(idx), spec.group, spec.head_dim)
        sub.prepare()
        qi = torch.from_numpy(idx).cuda()
        subs.append((sub, q[qi].contiguous(), torch.empty_like(q[qi])))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for sub, qq, oo in subs:
            P.packed_decode_step(sub, qq, oo, kernel=args.kernel)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for sub, qq, oo in subs:
                P.packed_decode_step(sub, qq, oo, kernel=args.kernel)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    n = max(10, min(args.steps, 100))
    st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for i in range(n):
        flush.zero_()
        st[i].record()
        g.replay()
        en[i].record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(st, en)) / n
    return {"ms_per_step": ms, "tok_s": spec.batch / (ms / 1e3), "launches_per_step": spec.layers,
            "note": "32 per-layer launches replayed from one CUDA graph"}


if __name__ == "__main__":
    main()
