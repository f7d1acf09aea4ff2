"""ctypes bindings shared by the C restatement (orc_*) and the reference shim (ref_*).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librdkv_ref.so")

# eps tables of proj/tests/fixtures/eps_reference.json (LLaMA-3.1-8B calibration)
EPS_V = {0: 1.0, 2: 0.313, 4: 0.014, 8: 4.9e-05, 16: 0.0}
EPS_K = {0: 1.0, 2: 0.149, 4: 0.0062, 8: 2.2e-05, 16: 0.0}


class Config(C.Structure):
    """Layout-identical to orc_config (oracle) and rdkv_config (include/rdkv_cuda.h)."""

    _fields_ = [
        ("n_tokens", C.c_int32),
        ("n_widths", C.c_int32),
        ("r_k", C.c_double),
        ("widths", C.c_int32 * 8),
        ("eps_v", C.c_double * 8),
        ("eps_k", C.c_double * 8),
        ("window", C.c_int32),
        ("pool_kernel", C.c_int32),
        ("tolerance", C.c_double),
        ("max_iterations", C.c_int32),
        ("strict_budget", C.c_int32),
        ("force_window_retain", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("lambda_v", C.c_double),
        ("lambda_k", C.c_double),
        ("objective_v", C.c_double),
        ("objective_k", C.c_double),
        ("achieved_bits", C.c_double),
        ("avg_v", C.c_double),
        ("avg_k", C.c_double),
        ("v_converged", C.c_int32),
        ("k_converged", C.c_int32),
        ("n_kept", C.c_int32),
        ("n_v16", C.c_int32),
        ("k_bits_len", C.c_int32),
        ("status", C.c_int32),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


def default_config(n_tokens=128, r_k=0.5, widths=(0, 2, 4, 8, 16), eps_v=None, eps_k=None,
                   window=32, pool_kernel=5, tolerance=1e-2, max_iterations=64,
                   strict_budget=False, force_window_retain=False) -> Config:
    """Reference defaults: pipeline.hpp:16-22, cache.hpp:29-34, allocator.hpp:12-19."""
    eps_v = eps_v or EPS_V
    eps_k = eps_k or EPS_K
    c = Config()
    c.n_tokens = n_tokens
    c.r_k = r_k
    c.n_widths = len(widths)
    for i, b in enumerate(widths):
        c.widths[i] = b
        c.eps_v[i] = eps_v[b]
        c.eps_k[i] = eps_k[b]
    c.window = window
    c.pool_kernel = pool_kernel
    c.tolerance = tolerance
    c.max_iterations = max_iterations
    c.strict_budget = int(strict_budget)
    c.force_window_retain = int(force_window_retain)
    return c


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: status {code}")
        self.code = code


F32 = C.POINTER(C.c_float)
F64 = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int)
I64 = C.POINTER(C.c_int64)
U8 = C.POINTER(C.c_uint8)


class TriZone:
    """Handle over orc_trizone / rdkv::TriZoneCache."""

    def __init__(self, lib: "OracleLib", handle, t_len, d):
        self._lib = lib
        self._h = handle
        self.t_len = t_len
        self.d = d

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib._fn("tz_free")(self._h)
            self._h = None

    @property
    def n_kept(self):
        return self._lib._fn("tz_n_kept")(self._h)

    def append(self, k, v):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        self._lib._check(self._lib._fn("tz_append")(self._h, _p(k, C.c_float), _p(v, C.c_float)),
                         "tz_append")

    def fused_logits(self, q):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(max(self.n_kept, 1), np.float64)
        self._lib._check(self._lib._fn("tz_fused_logits")(self._h, _p(q, C.c_float),
                                                          _p(out, C.c_double)), "fused_logits")
        return out[: self.n_kept]

    def decode(self, q):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(self.d, np.float64)
        self._lib._check(self._lib._fn("tz_decode")(self._h, _p(q, C.c_float),
                                                    _p(out, C.c_double)), "decode")
        return out

    def canon(self):
        n, d = self.n_kept, self.d
        nb = int(self._lib._fn("tz_payload_bytes")(self._h))
        kept = np.zeros(max(n, 1), np.int32)
        vcodes = np.zeros((max(n, 1), d), np.uint8)
        vscale = np.zeros(max(n, 1), np.float32)
        vzero = np.zeros(max(n, 1), np.int64)
        kcodes = np.zeros((d, max(n, 1)), np.uint8)
        kscale = np.zeros(d, np.float32)
        kzero = np.zeros(d, np.int64)
        vfp = np.zeros((max(n, 1), d), np.float32)
        kfp = np.zeros((max(n, 1), d), np.float32)
        payload = np.zeros(max(nb, 1), np.uint8)
        segtab = np.zeros((6, 6), np.int32)
        nseg = C.c_int()
        perm = np.zeros(d, np.int32)
        nperm = C.c_int()
        self._lib._check(self._lib._fn("tz_canon")(
            self._h, _p(kept, C.c_int), _p(vcodes, C.c_uint8), _p(vscale, C.c_float),
            _p(vzero, C.c_int64), _p(kcodes, C.c_uint8), _p(kscale, C.c_float),
            _p(kzero, C.c_int64), _p(vfp, C.c_float), _p(kfp, C.c_float), _p(payload, C.c_uint8),
            _p(segtab, C.c_int), C.byref(nseg), _p(perm, C.c_int), C.byref(nperm)), "canon")
        kcodes = kcodes[:, :n] if n else np.zeros((d, 0), np.uint8)
        return {
            "kept": kept[:n], "vcodes": vcodes[:n], "vscale": vscale[:n], "vzero": vzero[:n],
            "kcodes": np.ascontiguousarray(kcodes), "kscale": kscale, "kzero": kzero,
            "vfp": vfp[:n], "kfp": kfp[:n], "payload": payload[:nb],
            "segtab": segtab[: nseg.value], "perm": perm[: nperm.value],
        }


class OracleLib:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        self.kind = "reference" if prefix == "ref_" else "port"
        self._setup()

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    @staticmethod
    def _check(code, what):
        if code != 0:
            raise OracleError(code, what)

    def _setup(self):
        L = self.lib
        p = self.prefix
        getattr(L, p + "gen_synthetic").argtypes = [C.c_uint64] + [C.c_int] * 7 + [C.c_double, F32, F32, F32]
        getattr(L, p + "attention_probe").argtypes = [F32, C.c_int, F32, C.c_int, C.c_int, I32, F64]
        getattr(L, p + "moving_average").argtypes = [F32, C.c_int, C.c_int, F32]
        getattr(L, p + "channel_weights").argtypes = [F32, C.c_int, F32, C.c_int, C.c_int, F32]
        getattr(L, p + "quantize_unit").argtypes = [F32, C.c_int, C.c_int, U8, F32, I64]
        getattr(L, p + "mckp_bisect").argtypes = [F32, C.c_int, I32, F64, C.c_int, C.c_double,
                                                  C.c_double, C.c_int, C.c_int, I32, F64, F64, F64, I32]
        getattr(L, p + "allocate_head").argtypes = [F32, F32] + [C.c_int] * 5 + [
            C.POINTER(Config), I32, I32, F32, F32, C.POINTER(Stats)]
        getattr(L, p + "tz_build").argtypes = [F32, F32, C.c_int, C.c_int, I32, I32, I32]
        getattr(L, p + "tz_build").restype = C.c_void_p
        getattr(L, p + "tz_free").argtypes = [C.c_void_p]
        getattr(L, p + "tz_free").restype = None
        getattr(L, p + "tz_append").argtypes = [C.c_void_p, F32, F32]
        getattr(L, p + "tz_fused_logits").argtypes = [C.c_void_p, F32, F64]
        getattr(L, p + "tz_decode").argtypes = [C.c_void_p, F32, F64]
        getattr(L, p + "tz_n_kept").argtypes = [C.c_void_p]
        getattr(L, p + "tz_payload_bytes").argtypes = [C.c_void_p]
        getattr(L, p + "tz_payload_bytes").restype = C.c_size_t
        getattr(L, p + "tz_canon").argtypes = [C.c_void_p, I32, U8, F32, I64, U8, F32, I64, F32, F32,
                                               U8, I32, I32, I32, I32]
        if p == "ref_":
            L.ref_model_build.argtypes = [F32, F32, F32] + [C.c_int] * 6 + [
                C.POINTER(Config), F64, F64, I32]
            L.ref_model_build.restype = C.c_void_p
            L.ref_model_free.argtypes = [C.c_void_p]
            L.ref_model_free.restype = None
            L.ref_model_head.argtypes = [C.c_void_p, C.c_int, C.c_int, I32, I32, F32, F32,
                                         C.POINTER(Stats)]
            L.ref_model_trizone.argtypes = [C.c_void_p, C.c_int, C.c_int]
            L.ref_model_trizone.restype = C.c_void_p
            L.ref_model_decode.argtypes = [C.c_void_p, F32, F64, F64]
            L.ref_calibrate.argtypes = [F32, F32, F32] + [C.c_int] * 8 + [I32, C.c_int, F64,
                                                                        C.POINTER(C.c_longlong)]
            L.ref_run_sweep.argtypes = [F32, F32, F32] + [C.c_int] * 7 + [F64, C.c_int, C.POINTER(Config), F64]
            L.ref_save_cache.argtypes = [C.c_uint64] + [C.c_int] * 6 + [C.c_char_p]
            L.ref_load_cache.argtypes = [C.c_char_p, I32]
        else:
            L.orc_normal_stream.argtypes = [C.c_uint64, F32, C.c_size_t]
            L.orc_normal_stream.restype = None
            L.orc_dense_decode.argtypes = [F32, F32, F32, C.c_int, C.c_int, F64]
            L.orc_pack_bits.argtypes = [U8, C.c_int, C.c_int, U8]
            L.orc_head_budget.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int, F64, F64, F64, I32]
            L.orc_per_unit_argmin.argtypes = [C.c_double, I32, F64, C.c_int, C.c_double]
            L.orc_gen_counter.argtypes = [F32, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                          C.c_int, C.c_int, C.c_float, C.c_int, C.c_float]
            L.orc_gen_counter.restype = None

    # ---- API ---------------------------------------------------------------
    def gen_synthetic(self, seed, layers, q_heads, kv_heads, d, t_len, probe_window,
                      outlier_channels=0, outlier_scale=1.0):
        k = np.zeros((layers, kv_heads, t_len, d), np.float32)
        v = np.zeros_like(k)
        q = np.zeros((layers, q_heads, probe_window, d), np.float32)
        self._check(self._fn("gen_synthetic")(seed, layers, q_heads, kv_heads, d, t_len, probe_window,
                                              outlier_channels, outlier_scale, _p(k, C.c_float),
                                              _p(v, C.c_float), _p(q, C.c_float)), "gen_synthetic")
        return k, v, q

    def save_cache(self, seed, layers, q_heads, kv_heads, d, t_len, probe_window, path):
        """save_cache_file(gen_synthetic_cache(...)) (cache.cpp:205-226); reference only."""
        self._check(self.lib.ref_save_cache(seed, layers, q_heads, kv_heads, d, t_len, probe_window,
                                            path.encode()), "save_cache")

    def calibrate(self, k, v, q, granularity, widths):
        """calibrate_epsilon (quantizer.cpp:200-284) over caches k, v [n][L][H_kv][T][d],
        q [n][L][H_q][S_w][d]; returns (eps [n_widths], unit_count). Reference only."""
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        n, L, Hkv, T, d = k.shape
        Hq, Sw = q.shape[2], q.shape[3]
        w = np.ascontiguousarray(widths, np.int32)
        eps = np.zeros(len(w), np.float64)
        units = C.c_longlong(0)
        self._check(self.lib.ref_calibrate(_p(k, C.c_float), _p(v, C.c_float), _p(q, C.c_float), n, L, Hq,
                                           Hkv, d, T, Sw, granularity, _p(w, C.c_int), len(w),
                                           _p(eps, C.c_double), C.byref(units)), "calibrate")
        return eps, units.value

    def run_sweep(self, k, v, q, grid, cfg):
        """run_sweep (sweep.cpp:40-114) over caches k, v [n][L][H_kv][T][d], q [n][L][H_q][S_w][d];
        rows [n*len(grid)][5] = (seq_id, avg_bits, primal, dual, feasible). Reference only."""
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        n, L, Hkv, T, d = k.shape
        Hq, Sw = q.shape[2], q.shape[3]
        g = np.ascontiguousarray(grid, np.float64)
        if not isinstance(cfg, Config):
            cfg = Config.from_buffer_copy(bytes(cfg))  # same layout (test_struct_layouts_match_oracle)
        rows = np.zeros((n * len(g), 5), np.float64)
        self._check(self.lib.ref_run_sweep(_p(k, C.c_float), _p(v, C.c_float), _p(q, C.c_float), n, L, Hq, Hkv,
                                           d, T, Sw, _p(g, C.c_double), len(g), C.byref(cfg),
                                           _p(rows, C.c_double)), "run_sweep")
        return rows

    def load_cache_status(self, path):
        """(status, dims) of load_cache_file (cache.cpp:228-287); reference only."""
        dims = np.zeros(6, np.int32)
        code = self.lib.ref_load_cache(path.encode(), _p(dims, C.c_int32))
        return code, dims

    def attention_probe(self, q, k, offsets):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        offsets = np.ascontiguousarray(offsets, np.int32)
        a = np.zeros((q.shape[0], k.shape[0]), np.float64)
        self._check(self._fn("attention_probe")(_p(q, C.c_float), q.shape[0], _p(k, C.c_float),
                                                k.shape[0], k.shape[1], _p(offsets, C.c_int),
                                                _p(a, C.c_double)), "attention_probe")
        return a

    def moving_average(self, raw, kernel):
        raw = np.ascontiguousarray(raw, np.float32)
        out = np.zeros_like(raw)
        self._check(self._fn("moving_average")(_p(raw, C.c_float), raw.size, kernel,
                                               _p(out, C.c_float)), "moving_average")
        return out

    def channel_weights(self, q, k):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        out = np.zeros(q.shape[1], np.float32)
        self._check(self._fn("channel_weights")(_p(q, C.c_float), q.shape[0], _p(k, C.c_float),
                                                k.shape[0], q.shape[1], _p(out, C.c_float)),
                    "channel_weights")
        return out

    def quantize_unit(self, values, bits):
        values = np.ascontiguousarray(values, np.float32)
        codes = np.zeros(max(values.size, 1), np.uint8)
        scale = C.c_float()
        zp = C.c_int64()
        self._check(self._fn("quantize_unit")(_p(values, C.c_float), values.size, bits,
                                              _p(codes, C.c_uint8), C.byref(scale), C.byref(zp)),
                    "quantize_unit")
        return codes[: values.size], np.float32(scale.value), int(zp.value)

    def mckp_bisect(self, w, widths, eps, target, tolerance=1e-2, max_iterations=64,
                    strict_budget=False):
        w = np.ascontiguousarray(w, np.float32)
        widths = np.ascontiguousarray(widths, np.int32)
        eps = np.ascontiguousarray(eps, np.float64)
        bits = np.zeros(max(w.size, 1), np.int32)
        lam, avg, obj = C.c_double(), C.c_double(), C.c_double()
        conv = C.c_int()
        self._check(self._fn("mckp_bisect")(_p(w, C.c_float), w.size, _p(widths, C.c_int),
                                            _p(eps, C.c_double), widths.size, target, tolerance,
                                            max_iterations, int(strict_budget), _p(bits, C.c_int),
                                            C.byref(lam), C.byref(avg), C.byref(obj), C.byref(conv)),
                    "mckp_bisect")
        return {"bits": bits[: w.size], "lambda": lam.value, "avg": avg.value,
                "objective": obj.value, "converged": bool(conv.value)}

    def allocate_head(self, k_head, probe_group, kv_heads, cfg: Config):
        """k_head [T, d]; probe_group [g, probe_rows, d]."""
        k_head = np.ascontiguousarray(k_head, np.float32)
        probe_group = np.ascontiguousarray(probe_group, np.float32)
        t_len, d = k_head.shape
        g, rows, _ = probe_group.shape
        v_bits = np.zeros(t_len, np.int32)
        k_bits = np.zeros(d, np.int32)
        vw = np.zeros(t_len, np.float32)
        kw = np.zeros(d, np.float32)
        st = Stats()
        self._check(self._fn("allocate_head")(_p(k_head, C.c_float), _p(probe_group, C.c_float),
                                              t_len, d, g, rows, kv_heads, C.byref(cfg),
                                              _p(v_bits, C.c_int), _p(k_bits, C.c_int),
                                              _p(vw, C.c_float), _p(kw, C.c_float), C.byref(st)),
                    "allocate_head")
        s = st.as_dict()
        return {"v_bits": v_bits, "k_bits": k_bits[: s["k_bits_len"]], "v_weights": vw,
                "k_weights": kw, **s}

    def tz_build(self, k, v, v_bits, k_bits):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        v_bits = np.ascontiguousarray(v_bits, np.int32)
        t_len, d = k.shape
        kb = None if k_bits is None or len(k_bits) == 0 else np.ascontiguousarray(k_bits, np.int32)
        st = C.c_int()
        h = self._fn("tz_build")(_p(k, C.c_float), _p(v, C.c_float), t_len, d, _p(v_bits, C.c_int),
                                 _p(kb, C.c_int) if kb is not None else None, C.byref(st))
        if not h:
            raise OracleError(st.value, "tz_build")
        return TriZone(self, h, t_len, d)

    # oracle-only helpers
    def gen_counter(self, seed, tensor, first, count, d, seq_len, outlier_channels=0,
                    outlier_scale=1.0, hh_stride=0, hh_boost=0.0):
        """K0 values (FP16-representable float32), same as csrc/generate.cu."""
        out = np.empty(count, np.float32)
        self.lib.orc_gen_counter(_p(out, C.c_float), seed, tensor, first, count, d, seq_len,
                                 outlier_channels, outlier_scale, hh_stride, hh_boost)
        return out

    def normal_stream(self, seed, n):
        out = np.zeros(n, np.float32)
        self.lib.orc_normal_stream(seed, _p(out, C.c_float), n)
        return out

    def dense_decode(self, q, k_rows, v_rows):
        q = np.ascontiguousarray(q, np.float32)
        k_rows = np.ascontiguousarray(k_rows, np.float32)
        v_rows = np.ascontiguousarray(v_rows, np.float32)
        out = np.zeros(q.size, np.float64)
        self._check(self.lib.orc_dense_decode(_p(q, C.c_float), _p(k_rows, C.c_float),
                                              _p(v_rows, C.c_float), k_rows.shape[0], q.size,
                                              _p(out, C.c_double)), "dense_decode")
        return out

    def head_budget(self, n_tokens, r_k, head_dim, kv_heads):
        hb, vb, kb = C.c_double(), C.c_double(), C.c_double()
        sub = C.c_int()
        self._check(self.lib.orc_head_budget(n_tokens, r_k, head_dim, kv_heads, C.byref(hb),
                                             C.byref(vb), C.byref(kb), C.byref(sub)), "head_budget")
        return {"head_bits": hb.value, "v_bits": vb.value, "k_bits": kb.value, "sub_token": bool(sub.value)}

    def pack_bits(self, codes, bits):
        codes = np.ascontiguousarray(codes, np.uint8)
        per = 8 // bits
        out = np.zeros((codes.size + per - 1) // per, np.uint8)
        self._check(self.lib.orc_pack_bits(_p(codes, C.c_uint8), codes.size, bits,
                                           _p(out, C.c_uint8)), "pack_bits")
        return out

    def per_unit_argmin(self, weight, widths, eps, lam):
        widths = np.ascontiguousarray(widths, np.int32)
        eps = np.ascontiguousarray(eps, np.float64)
        r = self.lib.orc_per_unit_argmin(weight, _p(widths, C.c_int), _p(eps, C.c_double),
                                         widths.size, lam)
        if r < 0:
            raise OracleError(-r, "per_unit_argmin")
        return r


class RefModel:
    """allocate_model + build_packed_model + packed_decode_step via the reference (ref_ only)."""

    def __init__(self, lib: OracleLib, k, v, q, cfg: Config):
        self.lib = lib
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        self.layers, self.kv_heads, self.t_len, self.d = k.shape
        self.q_heads = q.shape[1]
        self.probe_rows = q.shape[2]
        a, p = C.c_double(), C.c_double()
        st = C.c_int()
        self._h = lib.lib.ref_model_build(_p(k, C.c_float), _p(v, C.c_float), _p(q, C.c_float),
                                          self.layers, self.q_heads, self.kv_heads, self.d,
                                          self.t_len, self.probe_rows, C.byref(cfg), C.byref(a),
                                          C.byref(p), C.byref(st))
        if not self._h:
            raise OracleError(st.value, "ref_model_build")
        self.alloc_seconds = a.value
        self.pack_seconds = p.value

    def __del__(self):
        if getattr(self, "_h", None):
            self.lib.lib.ref_model_free(self._h)
            self._h = None

    def head(self, layer, head):
        v_bits = np.zeros(self.t_len, np.int32)
        k_bits = np.zeros(self.d, np.int32)
        vw = np.zeros(self.t_len, np.float32)
        kw = np.zeros(self.d, np.float32)
        st = Stats()
        OracleLib._check(self.lib.lib.ref_model_head(self._h, layer, head, _p(v_bits, C.c_int),
                                                     _p(k_bits, C.c_int), _p(vw, C.c_float),
                                                     _p(kw, C.c_float), C.byref(st)), "model_head")
        s = st.as_dict()
        return {"v_bits": v_bits, "k_bits": k_bits[: s["k_bits_len"]], "v_weights": vw,
                "k_weights": kw, **s}

    def trizone(self, layer, head) -> TriZone:
        h = self.lib.lib.ref_model_trizone(self._h, layer, head)
        return _Borrowed(self.lib, h, self.t_len, self.d, self)

    def decode(self, q):
        """q [layers, q_heads, d] -> (out float64 same shape, seconds)."""
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(q.shape, np.float64)
        secs = C.c_double()
        OracleLib._check(self.lib.lib.ref_model_decode(self._h, _p(q, C.c_float),
                                                       _p(out, C.c_double), C.byref(secs)),
                         "model_decode")
        return out, secs.value


class _Borrowed(TriZone):
    def __init__(self, lib, handle, t_len, d, owner):
        super().__init__(lib, handle, t_len, d)
        self._owner = owner

    def __del__(self):
        self._h = None


def build(quiet=True) -> None:
    """Build liboracle.so and (when /root/reference exists) _ref/librdkv_ref.so."""
    cmd = ["make", "-C", HERE, "-j8", ORACLE_SO]
    if os.path.isdir("/root/reference/proj/core/src"):
        cmd.append("ref")
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL if quiet else None)


def load() -> OracleLib:
    if not os.path.exists(ORACLE_SO):
        build()
    return OracleLib(ORACLE_SO, "orc_")


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def load_ref() -> OracleLib:
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
    return OracleLib(REF_SO, "ref_")
