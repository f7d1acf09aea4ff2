"""Builds a packed multi-sequence, multi-layer decode workload on the device.

Every (sequence, layer) chunk of KV heads is generated on the device by K0,
run through weights -> allocate -> pack, and its tiles appended to one arena
(one unit per (sequence, layer, KV head), unit = (b * L + l) * H_kv + h), so a
single decode launch covers the whole step. Prefill-time work only; nothing
here runs inside a timed decode step.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import pipeline as P


def chunk_seed(base: int, seq: int, layer: int) -> int:
    """K0 seed of one (global sequence id, layer): the job is the same whatever
    the world size; a rank only picks which sequences it owns (dist.weak_shard)."""
    return (base * 1_000_003 + seq * 131 + layer) & ((1 << 63) - 1)


@dataclass
class WorkloadSpec:
    batch: int = 16
    layers: int = 32
    q_heads: int = 32
    kv_heads: int = 8
    head_dim: int = 128
    ctx: int = 131072
    probe_rows: int = 32
    n_tokens: int = 128
    seed: int = 1
    rank: int = 0
    hh_stride: int = 0      # heavy hitters (0 = plain Gaussian, like gen_synthetic_cache)
    hh_boost: float = 0.0
    outlier_channels: int = 0
    outlier_scale: float = 1.0
    zc_cap: int = 0
    # multi-GPU partition (north_star "by batch and KV head"):
    #   "seqs":  weak scaling, rank r owns sequences r*batch .. r*batch+batch-1, all KV heads
    #   "heads": strong scaling, every rank holds all `batch` sequences and its own
    #            contiguous range of KV heads (dist.strong_shard over kv_heads)
    shard: str = "seqs"
    world: int = 1

    def __post_init__(self):
        if self.shard not in ("seqs", "heads"):
            raise ValueError(f"shard must be 'seqs' or 'heads', not {self.shard!r}")
        if self.shard == "heads" and self.world > self.kv_heads:
            raise ValueError(f"cannot split {self.kv_heads} KV heads over {self.world} ranks")

    @property
    def first_seq(self):
        """Global id of this rank's first sequence (weak scaling: batch sequences per rank)."""
        return self.rank * self.batch if self.shard == "seqs" else 0

    @property
    def head_range(self) -> range:
        """Global KV heads this rank owns."""
        if self.shard == "seqs":
            return range(self.kv_heads)
        from .dist import strong_shard

        return strong_shard(self.kv_heads, self.rank, self.world).items

    @property
    def local_heads(self) -> int:
        return len(self.head_range)

    def global_unit(self, b: int, layer: int, h_local: int) -> int:
        """Unit id of (local sequence b, layer, local head) in the whole job
        ((seq * L + l) * H_kv + h, the reference's l * H_kv + h per sequence)."""
        return ((self.first_seq + b) * self.layers + layer) * self.kv_heads + self.head_range[h_local]

    @property
    def group(self):
        return self.q_heads // self.kv_heads

    @property
    def units(self):
        return self.batch * self.layers * self.local_heads


def gen_chunk(spec: WorkloadSpec, b: int, layer: int, dtype=torch.float16):
    """K, V [h, T, d] and probe Q [h, g, S_w, d] of one (sequence, layer), for the
    rank's h KV heads: the counter-based generator makes a head subset the exact
    slice of the full (sequence, layer) tensors (first_index offsets)."""
    s = chunk_seed(spec.seed, spec.first_seq + b, layer)
    T, d, g, Sw = spec.ctx, spec.head_dim, spec.group, spec.probe_rows
    h0, H = spec.head_range.start, spec.local_heads
    k = P.generate((H, T, d), dtype, seed=s, tensor=0, first_index=h0 * T * d, seq_len=T,
                   outlier_channels=spec.outlier_channels, outlier_scale=spec.outlier_scale,
                   hh_stride=spec.hh_stride, hh_boost=spec.hh_boost)
    v = P.generate((H, T, d), dtype, seed=s, tensor=1, first_index=h0 * T * d, seq_len=T)
    q = P.generate((H, g, Sw, d), dtype, seed=s, tensor=2, first_index=h0 * g * Sw * d, seq_len=T,
                   hh_stride=spec.hh_stride)
    return k, v, q


def build(spec: WorkloadSpec, cfg=None, log=None):
    """Returns (PackedModel over all units, timing dict, per-chunk allocation stats)."""
    cfg = cfg or P.default_config(n_tokens=spec.n_tokens, window=spec.probe_rows)
    chunks = []
    t_alloc = t_pack = t_gen = 0.0
    stats = []
    first_alloc = None
    for b in range(spec.batch):
        for layer in range(spec.layers):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            k, v, q = gen_chunk(spec, b, layer)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            # head budget over the model's KV heads (head_budget, pipeline.cpp:60-72),
            # whatever subset of them this rank holds
            alloc = P.allocate_model(k, q, cfg, kv_heads=spec.kv_heads)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            model = P.build_packed_model(k, v, alloc, group=spec.group)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            t_gen += t1 - t0
            t_alloc += t2 - t1
            t_pack += t3 - t2
            st = alloc.stats_host()
            if np.any(st["status"]):
                alloc.check()
            model.check()
            stats.append(st)
            if first_alloc is None:
                first_alloc = (alloc.v_bits.cpu().numpy(), alloc.k_bits.cpu().numpy(), st)
            chunks.append((model.arena[: model.arena_bytes], model.offsets_host))
            del k, v, q, alloc
    total = sum(int(o[-1]) for _, o in chunks)
    arena = torch.empty(total + 256, dtype=torch.uint8, device="cuda")
    offsets = np.zeros(spec.units + 1, np.int64)
    pos = 0
    u = 0
    for a, o in chunks:
        n = len(o) - 1
        arena[pos:pos + int(o[-1])] = a
        offsets[u:u + n] = o[:-1] + pos
        pos += int(o[-1])
        u += n
    offsets[u] = pos
    model = P.PackedModel(arena, torch.from_numpy(offsets).cuda(), offsets, spec.units, spec.group,
                          spec.head_dim)
    model.prepare()
    if spec.zc_cap:
        model.zc_k = torch.zeros((spec.units, spec.zc_cap, spec.head_dim), dtype=torch.float16, device="cuda")
        model.zc_v = torch.zeros_like(model.zc_k)
        model.zc_len = torch.zeros(spec.units, dtype=torch.int32, device="cuda")
        model.zc_cap = spec.zc_cap
    timing = {"gen_s": t_gen, "weights_alloc_s": t_alloc, "pack_s": t_pack}
    return model, timing, stats, first_alloc
