"""Device-resident RDKV pipeline over the C-ABI (allocate -> pack -> decode).

Python mirror of the reference's entry points for this path, batched over
units (one unit = one (batch, layer, KV head)):

    compute_weights     attention_probe + token/channel weights (pipeline.cpp:124-146)
    allocate            allocate_v + allocate_k via mckp_bisect (pipeline.cpp:74-112)
    allocate_model      both of the above (pipeline.cpp:191-207)
    build_packed_model  build_trizone for every unit (trizone.cpp:478-490)
    packed_decode_step  packed decode for every (unit, query head) (trizone.cpp:251-305)
    append_new_token    Zone C append (trizone.cpp:307-314)

torch supplies device memory and the current stream only; all compute runs in
the native sm_100a kernels of _lib/librdkv_b200.so.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import capi
from .capi import raise_for

EPS_V = {0: 1.0, 2: 0.313, 4: 0.014, 8: 4.9e-05, 16: 0.0}
EPS_K = {0: 1.0, 2: 0.149, 4: 0.0062, 8: 2.2e-05, 16: 0.0}

HEAD_STATS_DTYPE = np.dtype([
    ("lambda_v", "<f8"), ("lambda_k", "<f8"), ("objective_v", "<f8"), ("objective_k", "<f8"),
    ("achieved_bits", "<f8"), ("avg_v", "<f8"), ("avg_k", "<f8"), ("v_converged", "<i4"),
    ("k_converged", "<i4"), ("n_kept", "<i4"), ("n_v16", "<i4"), ("k_bits_len", "<i4"),
    ("status", "<i4"),
])
assert HEAD_STATS_DTYPE.itemsize == capi.HEAD_STATS_BYTES


def default_config(n_tokens=128, r_k=0.5, widths=(0, 2, 4, 8, 16), eps_v=None, eps_k=None,
                   window=32, pool_kernel=5, tolerance=1e-2, max_iterations=64,
                   strict_budget=False, force_window_retain=False) -> capi.Config:
    """Reference defaults (pipeline.hpp:16-22, cache.hpp:29-34, allocator.hpp:12-19)."""
    eps_v = eps_v or EPS_V
    eps_k = eps_k or EPS_K
    c = capi.Config()
    c.n_tokens, c.r_k, c.n_widths = n_tokens, r_k, len(widths)
    for i, b in enumerate(widths):
        c.widths[i], c.eps_v[i], c.eps_k[i] = b, eps_v[b], eps_k[b]
    c.window, c.pool_kernel = window, pool_kernel
    c.tolerance, c.max_iterations = tolerance, max_iterations
    c.strict_budget, c.force_window_retain = int(strict_budget), int(force_window_retain)
    return c


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return capi.RDKV_F32
    if t.dtype == torch.float16:
        return capi.RDKV_F16
    raise capi.InvalidArgument(capi.RDKV_EINVAL, f"unsupported dtype {t.dtype}")


def _check_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise capi.InvalidArgument(capi.RDKV_EINVAL, "tensors must be contiguous CUDA tensors")


def make_shape(units, seq_len, head_dim, group, probe_rows, kv_heads) -> capi.Shape:
    return capi.Shape(units, seq_len, head_dim, group, probe_rows, kv_heads)


# ---- K0 ---------------------------------------------------------------------
def generate(shape, dtype=torch.float16, seed=1, tensor=0, first_index=0, seq_len=None,
             outlier_channels=0, outlier_scale=1.0, hh_stride=0, hh_boost=0.0, device="cuda"):
    """Counter-based synthetic values (see csrc/generate.cu). shape[-1] = head_dim."""
    out = torch.empty(shape, dtype=dtype, device=device)
    d = shape[-1]
    t_len = seq_len or (shape[-2] if len(shape) >= 2 else 1)
    raise_for(capi.lib().rdkv_cuda_generate(
        out.data_ptr(), _dtype_code(out), seed, tensor, first_index, out.numel(), d, t_len,
        outlier_channels, float(outlier_scale), hh_stride, float(hh_boost), _stream()), "generate")
    return out


# ---- RDKVC001 containers -------------------------------------------------------
@dataclass
class DeviceCache:
    """KVCache (cache.hpp:90-107) resident on the device in unit order (unit = l*H_kv + h):
    k, v [U, T, d]; probe_q [U, g, S_w, d]."""

    k: torch.Tensor
    v: torch.Tensor
    probe_q: torch.Tensor
    layers: int
    q_heads: int
    kv_heads: int
    probe_window: int

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads


def read_cache_header(path: str) -> capi.CacheHeader:
    """Header of an RDKVC001 container, load_cache's checks (cache.cpp:228-287); host only."""
    h = capi.CacheHeader()
    raise_for(capi.lib().rdkv_cache_read_header(os.fsencode(path), C.byref(h)), f"load_cache_file({path})")
    return h


def load_cache_file(path: str, dtype=torch.float16, device="cuda") -> DeviceCache:
    """load_cache_file (cache.cpp:289-295) straight to device memory: the payload is streamed
    into k / v / probe_q in the container's own order (no host KVCache)."""
    h = read_cache_header(path)
    U, T, d = h.layers * h.kv_heads, h.seq_len, h.head_dim
    g = h.q_heads // h.kv_heads
    k = torch.empty((U, T, d), dtype=dtype, device=device)
    v = torch.empty_like(k)
    q = torch.empty((U, g, h.probe_window, d), dtype=dtype, device=device)
    raise_for(capi.lib().rdkv_cuda_cache_load(os.fsencode(path), C.byref(h), k.data_ptr(), v.data_ptr(),
                                              q.data_ptr(), _dtype_code(k), _stream()),
              f"load_cache_file({path})")
    return DeviceCache(k, v, q, h.layers, h.q_heads, h.kv_heads, h.probe_window)


# ---- ε calibration -------------------------------------------------------------
GRANULARITY = {"token": 0, "channel": 1}


def calibrate_epsilon(caches, granularity="token", widths=(0, 2, 4, 8, 16)):
    """calibrate_epsilon (quantizer.cpp:200-284) on the device: `caches` is a list of
    DeviceCache (or (k, v) pairs of [L*H_kv, T, d] device tensors). Token granularity
    calibrates on V rows, channel granularity on K columns. Returns (eps [n_widths] as a
    {width: eps} dict, unit_count); bit-identical to the reference for f32 inputs."""
    if not caches:
        raise capi.InvalidArgument(capi.RDKV_EINVAL, "calibrate_epsilon: empty sample")
    gran = GRANULARITY[granularity] if isinstance(granularity, str) else int(granularity)
    w = np.ascontiguousarray(widths, np.int32)
    nq = max(1, int(np.isin(w, (2, 4, 8)).sum()))
    L = capi.lib()
    sums, counts = [], []
    for c in caches:
        k, v = (c.k, c.v) if isinstance(c, DeviceCache) else c
        x = v if gran == 0 else k
        _check_cuda(x)
        x = x.contiguous()
        jobs, T, d = x.shape
        ws_bytes = L.rdkv_cuda_calibrate_workspace(jobs, T, d, gran, nq)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
        err = torch.empty((jobs, nq), dtype=torch.float64, device=x.device)
        cnt = torch.empty(jobs, dtype=torch.int64, device=x.device)
        raise_for(L.rdkv_cuda_calibrate_partials(x.data_ptr(), _dtype_code(x), jobs, T, d, gran,
                                                 w.ctypes.data, len(w), err.data_ptr(), cnt.data_ptr(),
                                                 ws.data_ptr(), ws_bytes, _stream()), "calibrate_epsilon")
        sums.append(err.cpu().numpy())
        counts.append(cnt.cpu().numpy())
    err_h = np.ascontiguousarray(np.concatenate(sums), np.float64)
    cnt_h = np.ascontiguousarray(np.concatenate(counts), np.int64)
    eps = np.zeros(len(w), np.float64)
    units = C.c_int64(0)
    raise_for(L.rdkv_calibrate_finalize(err_h.ctypes.data, cnt_h.ctypes.data, len(cnt_h), w.ctypes.data,
                                        len(w), eps.ctypes.data, C.byref(units)), "calibrate_epsilon")
    return {int(b): float(e) for b, e in zip(w, eps)}, int(units.value)


# ---- rate sweep with duality bounds -------------------------------------------
def mckp_bisect_batched(weights, widths, eps, target, tolerance=1e-2, max_iterations=64, strict=True):
    """mckp_bisect (allocator.cpp:135-216) over every row of weights [I, n] (device);
    returns (bits [I, n] u8, results [I] rdkv_bisect_result bytes, device)."""
    _check_cuda(weights)
    inst, n = weights.shape
    w = np.ascontiguousarray(widths, np.int32)
    e = np.ascontiguousarray(eps, np.float64)
    bits = torch.empty((inst, n), dtype=torch.uint8, device=weights.device)
    res = torch.empty(inst * C.sizeof(capi.BisectResult), dtype=torch.uint8, device=weights.device)
    raise_for(capi.lib().rdkv_cuda_mckp_bisect(weights.data_ptr(), inst, n, w.ctypes.data, e.ctypes.data, len(w),
                                               float(target), float(tolerance), int(max_iterations), int(strict),
                                               bits.data_ptr(), res.data_ptr(), _stream()), "mckp_bisect")
    return bits, res


def dual_bound_batched(weights, widths, eps, solved, total_budget):
    """dual_bound (allocator.cpp:218-246) of every row at its solved lambda (device)."""
    inst, n = weights.shape
    w = np.ascontiguousarray(widths, np.int32)
    e = np.ascontiguousarray(eps, np.float64)
    out = torch.empty(inst * C.sizeof(capi.DualBoundResult), dtype=torch.uint8, device=weights.device)
    raise_for(capi.lib().rdkv_cuda_dual_bound(weights.data_ptr(), inst, n, w.ctypes.data, e.ctypes.data, len(w),
                                              solved.data_ptr(), float(total_budget), out.data_ptr(), _stream()),
              "dual_bound")
    return out


def _structs(buf: torch.Tensor, ctype):
    raw = buf.cpu().numpy().tobytes()
    size = C.sizeof(ctype)
    return [ctype.from_buffer_copy(raw, i * size) for i in range(len(raw) // size)]


def run_sweep(caches, grid, cfg):
    """run_sweep (sweep.cpp:40-114) on the device: stage-1 weights once per cache, then per
    grid value a strict-budget bisection of every (layer, KV head) on both sides plus the dual
    bound at each final lambda; sums merge in head order on the host. `caches`: DeviceCache
    list. Returns rows (seq_id, avg_bits, primal, dual, feasible) ordered by (avg_bits, seq_id)."""
    grid = [float(b) for b in grid]
    if not grid:
        raise capi.InvalidArgument(capi.RDKV_EINVAL, "run_sweep: empty grid")
    if any(not (b > 0.0) or b > 16.0 for b in grid):
        raise capi.InvalidArgument(capi.RDKV_EINVAL, "run_sweep: grid values must be in (0, 16]")
    if cfg.window < 1 or cfg.pool_kernel < 1 or cfg.pool_kernel % 2 == 0:
        raise capi.InvalidArgument(capi.RDKV_EINVAL, "run_sweep: ProbeConfig")
    widths = [cfg.widths[i] for i in range(cfg.n_widths)]
    eps_v = [cfg.eps_v[i] for i in range(cfg.n_widths)]
    eps_k = [cfg.eps_k[i] for i in range(cfg.n_widths)]
    rows = []
    for seq, c in enumerate(caches):
        window = min(cfg.window, c.probe_window)
        w_t, w_c = compute_weights(c.k, c.probe_q, window=window, pool_kernel=cfg.pool_kernel,
                                   kv_heads=c.kv_heads)
        T, d = w_t.shape[1], w_c.shape[1]
        for target in grid:
            side = []
            for w, eps, n in ((w_t, eps_v, T), (w_c, eps_k, d)):
                _, res = mckp_bisect_batched(w, widths, eps, target, cfg.tolerance, cfg.max_iterations, True)
                db = dual_bound_batched(w, widths, eps, res, target * float(n))
                side.append((_structs(res, capi.BisectResult), _structs(db, capi.DualBoundResult)))
            primal = dual = 0.0
            feasible = True
            for (vr, vb), (kr, kb) in [((side[0][0][i], side[0][1][i]), (side[1][0][i], side[1][1][i]))
                                       for i in range(w_t.shape[0])]:
                for r in (vr, kr, vb, kb):
                    raise_for(r.status, "run_sweep")
                primal += vr.objective + kr.objective
                dual += vb.g_lambda + kb.g_lambda
                feasible = feasible and bool(vb.feasible) and bool(kb.feasible)
            rows.append((seq, target, primal, dual, feasible))
    rows.sort(key=lambda r: (r[1], r[0]))  # stable, like std::stable_sort
    return rows


# ---- K1 / K2 ----------------------------------------------------------------
def compute_weights(k: torch.Tensor, probe_q: torch.Tensor, window=32, pool_kernel=5,
                    kv_heads=1):
    """k [U, T, d]; probe_q [U, g, rows, d] -> (w_t [U, T] f32, w_c [U, d] f32)."""
    _check_cuda(k, probe_q)
    U, T, d = k.shape
    g, rows = probe_q.shape[1], probe_q.shape[2]
    shape = make_shape(U, T, d, g, rows, kv_heads)
    L = capi.lib()
    ws_bytes = L.rdkv_cuda_weights_workspace(C.byref(shape), window)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=k.device)
    w_t = torch.empty((U, T), dtype=torch.float32, device=k.device)
    w_c = torch.empty((U, d), dtype=torch.float32, device=k.device)
    raise_for(L.rdkv_cuda_weights(k.data_ptr(), probe_q.data_ptr(), _dtype_code(k), C.byref(shape),
                                  window, pool_kernel, w_t.data_ptr(), w_c.data_ptr(),
                                  ws.data_ptr(), ws_bytes, _stream()), "weights")
    return w_t, w_c


@dataclass
class Allocation:
    """Device ModelAllocation (pipeline.hpp:96-105) for U units."""

    v_bits: torch.Tensor          # [U, T] uint8
    k_bits: torch.Tensor          # [U, d] uint8
    stats: torch.Tensor           # [U * sizeof(rdkv_head_stats)] uint8
    w_t: torch.Tensor | None = None
    w_c: torch.Tensor | None = None

    def stats_host(self) -> np.ndarray:
        arr = np.frombuffer(self.stats.cpu().numpy().tobytes(), dtype=HEAD_STATS_DTYPE)
        return arr

    def check(self) -> None:
        st = self.stats_host()["status"]
        bad = np.nonzero(st)[0]
        if bad.size:
            raise_for(int(st[bad[0]]), f"allocate (unit {int(bad[0])})")


def allocate(w_t, w_c, cfg, group=1, probe_rows=32, kv_heads=1) -> Allocation:
    _check_cuda(w_t, w_c)
    U, T = w_t.shape
    d = w_c.shape[1]
    shape = make_shape(U, T, d, group, probe_rows, kv_heads)
    v_bits = torch.empty((U, T), dtype=torch.uint8, device=w_t.device)
    k_bits = torch.empty((U, d), dtype=torch.uint8, device=w_t.device)
    stats = torch.empty(U * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device=w_t.device)
    cfg = capi.config_from(cfg)
    raise_for(capi.lib().rdkv_cuda_allocate(w_t.data_ptr(), w_c.data_ptr(), C.byref(shape),
                                            C.byref(cfg), v_bits.data_ptr(), k_bits.data_ptr(),
                                            stats.data_ptr(), _stream()), "allocate")
    return Allocation(v_bits, k_bits, stats, w_t, w_c)


def allocate_model(k, probe_q, cfg, kv_heads) -> Allocation:
    """Stages 1-3 for every unit (allocate_model, pipeline.cpp:191-207)."""
    w_t, w_c = compute_weights(k, probe_q, window=cfg.window, pool_kernel=cfg.pool_kernel,
                               kv_heads=kv_heads)
    return allocate(w_t, w_c, cfg, group=probe_q.shape[1], probe_rows=probe_q.shape[2],
                    kv_heads=kv_heads)


# ---- K3 ---------------------------------------------------------------------
@dataclass
class PackedModel:
    """Device TriZone tiles of U units plus Zone C (PackedModel, trizone.hpp:128-136)."""

    arena: torch.Tensor
    offsets: torch.Tensor            # [U + 1] int64 (device)
    offsets_host: np.ndarray
    units: int
    group: int
    head_dim: int
    zc_k: torch.Tensor | None = None  # [U, cap, d] fp16
    zc_v: torch.Tensor | None = None
    zc_len: torch.Tensor | None = None  # [U] int32
    zc_cap: int = 0
    zc_count: int | None = 0  # host-side bound on every zc_len[u] (appends since packing); None = unknown
    head_status: torch.Tensor | None = None
    decode_sizes: torch.Tensor | None = None   # [U] int32, from prepare()
    plan: capi.DecodePlan | None = None
    unit_ids: torch.Tensor | None = None       # [U] int32: uniform-2-bit tiles first (split dispatch)
    split_ws: torch.Tensor | None = None       # split-K partials of the chunked mixed 2/4-bit kernel
    zc_ws: torch.Tensor | None = None          # Zone C prepass rows [U][g][d + 2] f32 (zc_workspace())
    _infos: list = field(default_factory=list)

    def prepare(self) -> capi.DecodePlan:
        """One-time tile scan enabling the tensor-core decode (rdkv_cuda_decode_prepare)."""
        offs = np.ascontiguousarray(self.offsets_host, np.int64)
        self.decode_sizes = torch.empty(self.units, dtype=torch.int32, device=self.arena.device)
        self.unit_ids = torch.empty(self.units, dtype=torch.int32, device=self.arena.device)
        plan = capi.DecodePlan()
        raise_for(capi.lib().rdkv_cuda_decode_prepare_split(self.arena.data_ptr(), offs.ctypes.data, self.units,
                                                            self.decode_sizes.data_ptr(), self.unit_ids.data_ptr(),
                                                            C.byref(plan), _stream()), "decode_prepare")
        self.plan = plan
        # long or mixed 2/4-bit tiles decode on the chunked split-K kernel (decode_u24),
        # whose parts' partials live in a caller-owned workspace (the library keeps no state)
        self.split_ws = None
        if plan.mix24 and not (plan.uniform2 and plan.max_slots <= 160):
            parts = min(16, int(plan.min_chunks24))
            if parts > 1:
                self.split_ws = decode_workspace(self, parts, self.arena.device)
        return plan

    def share_plan(self, other: "PackedModel") -> "PackedModel":
        """Reuse another model's prepare() results (same tiles, e.g. an arena copy)."""
        self.decode_sizes, self.plan, self.unit_ids = other.decode_sizes, other.plan, other.unit_ids
        self.split_ws = other.split_ws
        self.zc_ws = other.zc_ws
        return self

    def zc_workspace(self) -> torch.Tensor:
        """Scratch of the Zone C prepass (one [g][d + 2] f32 row set per unit): with it the
        short-tile decode folds the appended rows in without staging them (csrc/decode_mma.cu
        zc_partial_kernel); without it the fused / chunked Zone C variants run."""
        need = self.units * self.group * (self.head_dim + 2) * 4
        if self.zc_ws is None or self.zc_ws.numel() < need:
            self.zc_ws = torch.empty(need, dtype=torch.uint8, device=self.arena.device)
        return self.zc_ws

    @property
    def arena_bytes(self) -> int:
        return int(self.offsets_host[-1])

    def tile_bytes(self, unit: int) -> np.ndarray:
        a, b = int(self.offsets_host[unit]), int(self.offsets_host[unit + 1])
        return self.arena[a:b].cpu().numpy()

    def info(self, unit: int) -> capi.TileInfo:
        t = self.tile_bytes(unit)
        info = capi.TileInfo()
        raise_for(capi.lib().rdkv_tile_info_get(t.ctypes.data, C.byref(info)), "tile_info")
        return info

    def infos(self) -> list:
        """TileInfo of every unit (one bulk D2H copy of the arena)."""
        host = self.arena.cpu().numpy()
        out = []
        for u in range(self.units):
            info = capi.TileInfo()
            raise_for(capi.lib().rdkv_tile_info_get(host[int(self.offsets_host[u]):].ctypes.data,
                                                    C.byref(info)), "tile_info")
            out.append(info)
        return out

    def decode_bytes(self, io_bytes=2) -> int:
        """Algorithmic bytes of one decode step: every tile's decode region, Zone C
        rows, q and out."""
        tiles = sum(int(i.decode_bytes) for i in self.infos())
        zc = 0 if self.zc_len is None else int(self.zc_len.sum().item()) * self.head_dim * 2 * 2
        qo = self.units * self.group * self.head_dim * io_bytes * 2
        return tiles + zc + qo

    def survey_bytes(self, io_bytes=2) -> int:
        """SURVEY.md §8(d)'s algorithmic bytes of one decode step, from the
        allocation alone: K codes N_k (pad4(c2)/4 + pad2(c4)/2 + c8) + k16
        N_k c16 2 + V codes (r2 d/4 + r4 d/2 + r8 d) + Zone B r16 d 2 + params
        8 (r2 + r4 + r8) + 8 (c2 + c4 + c8) + channel map (d - c0) + Zone C
        + q and out. decode_bytes() minus this = the layout's own overhead
        (tile header, 16-bit perm entries, class padding)."""
        d = self.head_dim
        tot = 0
        for i in self.infos():
            n = int(i.n_kept)
            r2, r4, r8, r16 = (int(x) for x in i.rows)
            c2, c4, c8, c16 = (int(x) for x in i.chans)
            kq = n * ((c2 + 3) // 4 + (c4 + 1) // 2 + c8) + n * c16 * 2
            vq = r2 * d // 4 + r4 * d // 2 + r8 * d + r16 * d * 2
            tot += kq + vq + 8 * (r2 + r4 + r8) + 8 * (c2 + c4 + c8) + (c2 + c4 + c8 + c16)
        zc = 0 if self.zc_len is None else int(self.zc_len.sum().item()) * d * 2 * 2
        return tot + zc + self.units * self.group * d * io_bytes * 2

    def export(self, unit: int) -> dict:
        """Canonical reference view of one tile (see rdkv_tile_export)."""
        t = self.tile_bytes(unit)
        return export_tile(t, self.head_dim)

    def check(self) -> None:
        if self.head_status is None:
            return
        st = self.head_status.cpu().numpy()
        bad = np.nonzero(st)[0]
        if bad.size:
            raise_for(int(st[bad[0]]), f"pack (unit {int(bad[0])})")


def export_tile(tile: np.ndarray, d: int) -> dict:
    tile = np.ascontiguousarray(tile, np.uint8)
    L = capi.lib()
    info = capi.TileInfo()
    raise_for(L.rdkv_tile_info_get(tile.ctypes.data, C.byref(info)), "tile_info")
    n = int(info.n_kept)
    nb = int(L.rdkv_tile_export_payload_bytes(tile.ctypes.data, d))
    m = max(n, 1)
    kept = np.zeros(m, np.int32)
    vcodes = np.zeros((m, d), np.uint8)
    vscale = np.zeros(m, np.float32)
    vzero = np.zeros(m, np.int64)
    kcodes = np.zeros((d, m), np.uint8)
    kscale = np.zeros(d, np.float32)
    kzero = np.zeros(d, np.int64)
    vfp = np.zeros((m, d), np.float32)
    kfp = np.zeros((m, d), np.float32)
    payload = np.zeros(max(nb, 1), np.uint8)
    segtab = np.zeros((6, 6), np.int32)
    nseg = C.c_int32()
    perm = np.zeros(d, np.int32)
    nperm = C.c_int32()
    raise_for(L.rdkv_tile_export(tile.ctypes.data, d, kept.ctypes.data, vcodes.ctypes.data,
                                 vscale.ctypes.data, vzero.ctypes.data, kcodes.ctypes.data,
                                 kscale.ctypes.data, kzero.ctypes.data, vfp.ctypes.data,
                                 kfp.ctypes.data, payload.ctypes.data, segtab.ctypes.data,
                                 C.addressof(nseg), perm.ctypes.data, C.addressof(nperm)), "export")
    # kcodes was written channel-major with row stride n
    kc = kcodes.reshape(-1)[: d * n].reshape(d, n) if n else np.zeros((d, 0), np.uint8)
    return {"kept": kept[:n], "vcodes": vcodes[:n], "vscale": vscale[:n], "vzero": vzero[:n],
            "kcodes": kc, "kscale": kscale, "kzero": kzero, "vfp": vfp[:n], "kfp": kfp[:n],
            "payload": payload[:nb], "segtab": segtab[: nseg.value], "perm": perm[: nperm.value],
            "info": info}


def import_tile(d: int, kept, v_bits_kept, vcodes, vscale, vzero, vfp, k_bits, kcodes, kscale, kzero,
                kfp) -> np.ndarray:
    """Device tile bytes (host copy) from a reference TriZone view (rdkv_tile_import)."""
    L = capi.lib()
    n = len(kept)
    m = max(n, 1)

    def arr(x, dt, shape):
        a = np.zeros(shape, dt)
        x = np.asarray(x, dt)
        if x.size:
            a.reshape(-1)[: x.size] = x.reshape(-1)
        return a

    kept_a = arr(kept, np.int32, m)
    vb = arr(v_bits_kept, np.uint8, m)
    kb = arr(k_bits, np.uint8, d)
    vc = arr(vcodes, np.uint8, (m, d))
    vs = arr(vscale, np.float32, m)
    vz = arr(vzero, np.int64, m)
    vf = arr(vfp, np.float32, (m, d))
    kc = arr(kcodes, np.uint8, (d, m))  # channel-major, row stride n
    ks = arr(kscale, np.float32, d)
    kz = arr(kzero, np.int64, d)
    kf = arr(kfp, np.float32, (m, d))
    nbytes = int(L.rdkv_tile_import_bytes(d, n, vb.ctypes.data, kb.ctypes.data))
    if nbytes == 0:
        raise_for(capi.RDKV_EINVAL, "tile_import_bytes")
    tile = np.zeros(nbytes, np.uint8)
    raise_for(L.rdkv_tile_import(d, n, kept_a.ctypes.data, vb.ctypes.data, vc.ctypes.data, vs.ctypes.data,
                                 vz.ctypes.data, vf.ctypes.data, kb.ctypes.data, kc.ctypes.data, ks.ctypes.data,
                                 kz.ctypes.data, kf.ctypes.data, tile.ctypes.data, nbytes), "tile_import")
    return tile


def build_packed_model(k, v, alloc: Allocation, group, zc_cap=0) -> PackedModel:
    """build_trizone for every unit into one arena (trizone.cpp:478-490)."""
    _check_cuda(k, v)
    U, T, d = k.shape
    shape = make_shape(U, T, d, group, 1, 1)
    L = capi.lib()
    offsets = torch.empty(U + 1, dtype=torch.int64, device=k.device)
    raise_for(L.rdkv_cuda_pack_plan(alloc.v_bits.data_ptr(), alloc.k_bits.data_ptr(),
                                    C.byref(shape), offsets.data_ptr(), _stream()), "pack_plan")
    offsets_host = offsets.cpu().numpy()
    arena = torch.empty(int(offsets_host[-1]) + 256, dtype=torch.uint8, device=k.device)
    status = torch.zeros(U, dtype=torch.int32, device=k.device)
    raise_for(L.rdkv_cuda_pack(k.data_ptr(), v.data_ptr(), _dtype_code(k), alloc.v_bits.data_ptr(),
                               alloc.k_bits.data_ptr(), C.byref(shape), offsets.data_ptr(),
                               arena.data_ptr(), status.data_ptr(), _stream()), "pack")
    model = PackedModel(arena, offsets, offsets_host, U, group, d, head_status=status)
    model.prepare()
    if zc_cap > 0:
        model.zc_k = torch.zeros((U, zc_cap, d), dtype=torch.float16, device=k.device)
        model.zc_v = torch.zeros((U, zc_cap, d), dtype=torch.float16, device=k.device)
        model.zc_len = torch.zeros(U, dtype=torch.int32, device=k.device)
        model.zc_cap = zc_cap
    return model


# ---- K4 / K5 ----------------------------------------------------------------
def decode_args(model: PackedModel, q, out, split=1, kernel=0, workspace=None) -> capi.DecodeArgs:
    a = capi.DecodeArgs()
    a.arena = model.arena.data_ptr()
    a.tile_offsets = model.offsets.data_ptr()
    a.units, a.group, a.head_dim = model.units, model.group, model.head_dim
    a.io_dtype = _dtype_code(q)
    a.q, a.out = q.data_ptr(), out.data_ptr()
    if model.zc_len is not None:
        a.zc_k, a.zc_v, a.zc_len = model.zc_k.data_ptr(), model.zc_v.data_ptr(), model.zc_len.data_ptr()
        a.zc_cap = model.zc_cap
        if model.zc_count is not None:
            a.flags |= capi.RDKV_DECODE_ZC_BOUND
            a.zc_bound = min(model.zc_count, model.zc_cap)
    a.split = split
    a.kernel = kernel
    if model.plan is not None:
        a.tile_decode_bytes = model.decode_sizes.data_ptr()
        a.plan = model.plan
        if model.unit_ids is not None:
            a.unit_ids = model.unit_ids.data_ptr()
    if workspace is None and split == 1 and kernel in (0, 2) and model.split_ws is not None:
        a.split = 0  # automatic split-K over the model's partials workspace
        workspace = model.split_ws
    elif workspace is None and split == 1 and kernel in (0, 2) and model.zc_len is not None:
        workspace = model.zc_workspace()  # Zone C prepass rows (short uniform-2-bit tiles)
    if workspace is not None:
        a.workspace, a.workspace_bytes = workspace.data_ptr(), workspace.numel()
    return a


def decode_workspace(model: PackedModel, split: int, device="cuda"):
    n = capi.lib().rdkv_cuda_decode_workspace(model.units, model.group, model.head_dim, split)
    return torch.empty(max(n, 1), dtype=torch.uint8, device=device) if n else None


def packed_decode_step(model: PackedModel, q, out=None, split=1, kernel=0, workspace=None):
    """q [U, g, d] (f32 or f16) -> out, same shape/dtype (trizone.cpp:251-305)."""
    _check_cuda(q)
    if out is None:
        out = torch.empty_like(q)
    if split > 1 and workspace is None:
        workspace = decode_workspace(model, split, q.device)
    a = decode_args(model, q, out, split, kernel, workspace)
    raise_for(capi.lib().rdkv_cuda_decode(C.byref(a), _stream()), "decode")
    return out


def chunk_ranges(nslot: int) -> list[tuple[int, int]]:
    """Token-slot chunks of a tile in the chunked / sequence-split decode
    (u2c_geom in csrc/decode_mma.cu): <= 160 slots each, starts 32-aligned."""
    C = 1 if nslot <= 160 else (nslot + 159) // 160
    S = nslot if C == 1 else ((nslot + C - 1) // C + 31) & ~31
    return [(c * S, min(S, nslot - c * S)) for c in range(C)]


def decode_partial(model: PackedModel, q, rank: int, world: int, partial=None):
    """This rank's share of a sequence-split step (rdkv_cuda_decode_partial):
    token chunks c % world == rank of every tile -> [U, g, d + 2] f32
    (unnormalised o, running max in log2 units, weight sum)."""
    _check_cuda(q)
    U, g, d = model.units, model.group, model.head_dim
    if partial is None:
        partial = torch.empty((U, g, d + 2), dtype=torch.float32, device=q.device)
    a = decode_args(model, q, q, 1, 0)
    raise_for(capi.lib().rdkv_cuda_decode_partial(C.byref(a), rank, world, partial.data_ptr(), _stream()),
              "decode_partial")
    return partial


def merge_partials(parts, dtype=torch.float16, out=None):
    """[R, U, g, d + 2] partials -> out [U, g, d] (rdkv_cuda_decode_merge)."""
    _check_cuda(parts)
    R, U, g, d2 = parts.shape
    if out is None:
        out = torch.empty((U, g, d2 - 2), dtype=dtype, device=parts.device)
    raise_for(capi.lib().rdkv_cuda_decode_merge(parts.contiguous().data_ptr(), R, U, g, d2 - 2, out.data_ptr(),
                                                _dtype_code(out), _stream()), "decode_merge")
    return out


def merge_partials_reference(parts):
    """The merge in plain torch (any device): sum_r 2^(m_r - M) o_r / sum_r 2^(m_r - M) l_r."""
    o, m, l = parts[..., :-2].double(), parts[..., -2].double(), parts[..., -1].double()
    M = m.max(dim=0).values
    w = torch.where(l > 0, torch.exp2(m - M), torch.zeros_like(m))
    return (w.unsqueeze(-1) * o).sum(0) / (w * l).sum(0).unsqueeze(-1)


class HostDecoder:
    """End-to-end decode from pinned host q to pinned host out through the
    pipelined C-ABI entry point (rdkv_cuda_decode_host_pipelined): the step is
    cut into `chunks` unit ranges whose H2D copy, decode and D2H copy overlap.
    Owns the native context (two copy streams + events) and the device staging
    buffers; one step at a time per instance."""

    def __init__(self, model: PackedModel, dtype=torch.float16, chunks: int = 8, kernel: int = 0):
        self.model = model
        shape = (model.units, model.group, model.head_dim)
        self.q_dev = torch.empty(shape, dtype=dtype, device=model.arena.device)
        self.out_dev = torch.empty_like(self.q_dev)
        self.kernel = kernel
        ctx = C.c_void_p()
        raise_for(capi.lib().rdkv_cuda_decode_ctx_create(chunks, C.byref(ctx)), "decode_ctx_create")
        self.ctx = ctx

    def step(self, q_host: torch.Tensor, out_host: torch.Tensor, stream: int | None = None) -> None:
        """Enqueue one step on `stream` (default: torch's current stream)."""
        if q_host.dtype != self.q_dev.dtype or out_host.dtype != self.q_dev.dtype:
            raise capi.InvalidArgument(capi.RDKV_EINVAL, "host buffers must match the decoder dtype")
        if q_host.shape != self.q_dev.shape or out_host.shape != self.q_dev.shape:
            raise capi.InvalidArgument(capi.RDKV_EINVAL, "host buffers must be [units, group, head_dim]")
        raise_for(capi.lib().rdkv_cuda_decode_host_pipelined(self.ctx, C.byref(self.args), q_host.data_ptr(),
                                                             out_host.data_ptr(),
                                                             _stream() if stream is None else stream),
                  "decode_host_pipelined")

    @property
    def args(self) -> capi.DecodeArgs:
        """Decode arguments rebuilt from the model at every step: the Zone C bound
        (RDKV_DECODE_ZC_BOUND / zc_bound) follows the appends made since the last
        step, and a changed bound changes the native graph-cache key."""
        return decode_args(self.model, self.q_dev, self.out_dev, 1, self.kernel)

    def close(self) -> None:
        if getattr(self, "ctx", None):
            capi.lib().rdkv_cuda_decode_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def append_new_token(model: PackedModel, k_new, v_new) -> None:
    """One K/V row per unit into Zone C (trizone.cpp:307-314)."""
    if model.zc_len is None:
        raise capi.InvalidArgument(capi.RDKV_EINVAL, "model built without Zone C capacity")
    _check_cuda(k_new, v_new)
    # the reference appends without limit (trizone.cpp:307-314); the device Zone C
    # has a fixed capacity, so a full cache is an error instead of a dropped row
    full = (model.zc_count >= model.zc_cap if model.zc_count is not None
            else int(model.zc_len.max().item()) >= model.zc_cap)
    if full:
        raise capi.InvalidArgument(capi.RDKV_EINVAL,
                                   f"append_new_token: Zone C capacity {model.zc_cap} exhausted")
    raise_for(capi.lib().rdkv_cuda_append(model.zc_k.data_ptr(), model.zc_v.data_ptr(),
                                          model.zc_len.data_ptr(), model.zc_cap, k_new.data_ptr(),
                                          v_new.data_ptr(), _dtype_code(k_new), model.units,
                                          model.head_dim, _stream()), "append")
    if model.zc_count is not None:
        model.zc_count += 1
