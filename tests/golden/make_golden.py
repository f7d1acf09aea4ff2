"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs the compiled reference (oracle/_ref/librdkv_ref.so, built by
oracle/Makefile from /root/reference/proj/core/src) and records inputs and
outputs of the hot path: the synthetic generator, allocate_head, mckp_bisect,
build_trizone (canonical export incl. raw PackedSegment payload bytes) and
packed_decode_step. Re-run from the repo root:

    python tests/golden/make_golden.py

The fixtures travel to the GPU box; /root/reference does not.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

ref = oracle.load_ref()
orc = oracle.load()  # only its mt19937 stream helper is used (pinned by gen.npz)


def rng_tensor(rng, *shape):
    return rng.standard_normal(shape).astype(np.float32)


def canon_dict(prefix, c):
    return {f"{prefix}_{k}": np.asarray(v) for k, v in c.items()}


def make_gen():
    out = {}
    k, v, q = ref.gen_synthetic(1, 1, 4, 2, 16, 64, 16)
    out.update(k1=k, v1=v, q1=q)
    k, v, q = ref.gen_synthetic(7, 1, 2, 2, 32, 128, 32, 3, 100.0)
    out.update(k2=k, v2=v, q2=q)
    np.savez_compressed(os.path.join(HERE, "gen.npz"), **out)


ALLOC_CASES = [
    # (seed, (L, Hq, Hkv, d, T), S_w, outliers, scale, head, cfg kwargs)
    (99, (1, 4, 2, 16, 48), 16, 0, 1.0, 0, dict(n_tokens=48 * 2)),              # saturated: identity
    (7, (1, 2, 2, 32, 128), 32, 3, 100.0, 0, dict(n_tokens=32)),               # outlier channels
    (61, (1, 4, 2, 8, 32), 16, 0, 1.0, 1, dict(n_tokens=16, window=8)),        # narrow window
    (15, (1, 2, 2, 16, 64), 8, 0, 1.0, 0, dict(n_tokens=8, force_window_retain=True)),
    (33, (1, 4, 4, 32, 256), 32, 0, 1.0, 2, dict(n_tokens=256, strict_budget=True)),
    (21, (1, 4, 2, 16, 64), 16, 0, 1.0, 1, dict(n_tokens=24)),
    (5, (1, 8, 2, 64, 512), 32, 4, 8.0, 1, dict(n_tokens=512, r_k=0.4)),
    (11, (1, 4, 1, 16, 40), 16, 0, 1.0, 0, dict(n_tokens=1, window=16)),       # near-total eviction
]


def make_alloc():
    out = {"n": np.int32(len(ALLOC_CASES))}
    for i, (seed, (L, Hq, Hkv, d, T), sw, oc, osc, head, kw) in enumerate(ALLOC_CASES):
        k, v, q = ref.gen_synthetic(seed, L, Hq, Hkv, d, T, sw, oc, osc)
        g = Hq // Hkv
        cfg = oracle.default_config(**kw)
        r = ref.allocate_head(k[0, head], q[0, head * g:(head + 1) * g], Hkv, cfg)
        out[f"c{i}_k"] = k[0, head]
        out[f"c{i}_v"] = v[0, head]
        out[f"c{i}_q"] = q[0, head * g:(head + 1) * g]
        out[f"c{i}_kv_heads"] = np.int32(Hkv)
        cfgarr = np.frombuffer(bytes(cfg), dtype=np.uint8)
        out[f"c{i}_cfg"] = cfgarr
        for key in ("v_bits", "k_bits", "v_weights", "k_weights"):
            out[f"c{i}_{key}"] = np.asarray(r[key])
        for key in ("lambda_v", "lambda_k", "objective_v", "objective_k", "achieved_bits",
                    "v_converged", "k_converged", "n_kept", "n_v16", "k_bits_len"):
            out[f"c{i}_{key}"] = np.asarray(r[key])
        tz = ref.tz_build(k[0, head], v[0, head], r["v_bits"], r["k_bits"])
        out.update(canon_dict(f"c{i}_tz", tz.canon()))
    np.savez_compressed(os.path.join(HERE, "alloc.npz"), **out)


def make_trizone():
    rng = np.random.default_rng(1007)
    choices = np.array([0, 2, 4, 8, 16])
    out = {}
    shapes = [(13, 5), (64, 16), (64, 32), (40, 7), (256, 32), (24, 64), (9, 4), (64, 33),
              (100, 128), (16, 3), (48, 64), (200, 128)]
    for i, (T, d) in enumerate(shapes):
        k = rng_tensor(rng, T, d)
        v = rng_tensor(rng, T, d)
        if i == 7:
            v[3] = 5.0  # constant row: degenerate range (quantizer.cpp:117)
            k[:, 2] = -1.5  # constant column
        vb = choices[rng.integers(0, 5, T)].astype(np.int32)
        vb[rng.integers(0, T)] = 8
        kb = choices[rng.integers(0, 5, d)].astype(np.int32)
        if i == 9:
            kb[:] = 0  # every K channel removed: uniform attention
        if i == 10:
            vb[:] = 16
            kb[:] = 16  # identity compression
        tz = ref.tz_build(k, v, vb, kb)
        appends = int(rng.integers(0, 9))
        ak = rng_tensor(rng, max(appends, 1), d)
        av = rng_tensor(rng, max(appends, 1), d)
        for a in range(appends):
            tz.append(ak[a], av[a])
        qs = rng_tensor(rng, 4, d)
        outs = np.stack([tz.decode(qs[j]) for j in range(4)])
        fused = np.stack([np.pad(tz.fused_logits(qs[j]), (0, T - tz.n_kept)) for j in range(4)])
        out.update({f"t{i}_k": k, f"t{i}_v": v, f"t{i}_v_bits": vb, f"t{i}_k_bits": kb,
                    f"t{i}_appends": np.int32(appends), f"t{i}_ak": ak, f"t{i}_av": av,
                    f"t{i}_q": qs, f"t{i}_out": outs, f"t{i}_fused": fused})
        out.update(canon_dict(f"t{i}_tz", ref.tz_build(k, v, vb, kb).canon()))
    out["n"] = np.int32(len(shapes))
    np.savez_compressed(os.path.join(HERE, "trizone.npz"), **out)


def make_mckp():
    rng = np.random.default_rng(1010)
    out = {}
    n_cases = 40
    for i in range(n_cases):
        n = int(rng.integers(4, 1024)) if i % 4 else int(rng.integers(1, 12))
        w = (10.0 ** rng.uniform(-2.0, 2.0, n)).astype(np.float32)
        if i % 7 == 3:
            w[rng.integers(0, n, max(1, n // 5))] = 0.0
        e2 = 10 ** rng.uniform(-1.2, -0.3)
        e4 = e2 * 10 ** rng.uniform(-2.0, -1.0)
        e8 = e4 * 10 ** rng.uniform(-2.2, -1.2)
        widths = np.array([0, 2, 4, 8, 16], np.int32)
        eps = np.array([1.0, e2, e4, e8, 0.0])
        if i % 10 == 9:
            widths = np.array([2, 4, 8, 16], np.int32)
            eps = eps[1:]
        target = float(rng.uniform(0.05, 15.5)) if i % 9 else 16.0
        strict = bool(i % 3 == 0)
        r = ref.mckp_bisect(w, widths, eps, target, 1e-2, 64, strict)
        out.update({f"m{i}_w": w, f"m{i}_widths": widths, f"m{i}_eps": eps,
                    f"m{i}_target": np.float64(target), f"m{i}_strict": np.int32(strict),
                    f"m{i}_bits": r["bits"], f"m{i}_lambda": np.float64(r["lambda"]),
                    f"m{i}_avg": np.float64(r["avg"]), f"m{i}_objective": np.float64(r["objective"]),
                    f"m{i}_converged": np.int32(r["converged"])})
    out["n"] = np.int32(n_cases)
    np.savez_compressed(os.path.join(HERE, "mckp.npz"), **out)


def make_cache_io():
    """RDKVC001 containers (cache.cpp:205-287): one written by the reference's save_cache_file
    plus byte-level variants, each with the status + dims of the reference's load_cache_file."""
    import json
    import struct
    import tempfile
    tmp = tempfile.mkdtemp()
    base_path = os.path.join(tmp, "base.rdkvc")
    ref.save_cache(3, 2, 4, 2, 8, 16, 4, base_path)
    base = open(base_path, "rb").read()
    hlen = struct.unpack("<I", base[8:12])[0]
    htext = base[12:12 + hlen].decode()
    payload = base[12 + hlen:]
    hdr = json.loads(htext)

    def with_header(text, pl=payload):
        t = text.encode()
        return b"RDKVC001" + struct.pack("<I", len(t)) + t + pl

    def edit(**kw):
        h = dict(hdr)
        for k, v in kw.items():
            if v is None:
                h.pop(k)
            else:
                h[k] = v
        return with_header(json.dumps(h, separators=(",", ":")))

    nan_pl = bytearray(payload)
    kv_bytes = 2 * 2 * 16 * 8 * 4
    nan_pl[kv_bytes + 40:kv_bytes + 44] = struct.pack("<f", float("nan"))
    inf_pl = bytearray(payload)
    inf_pl[-4:] = struct.pack("<f", float("inf"))
    big_pl = bytearray(payload)
    big_pl[4:8] = struct.pack("<f", 1.0e6)
    variants = {
        "ok": base,
        "pretty_extra_keys": with_header(json.dumps(dict(hdr, note={"a": [1, 2.5, None, True]}), indent=2)),
        "float_dim": with_header(htext.replace('"d":8', '"d":8.0')),
        "bad_magic": b"RDKVC002" + base[8:],
        "short_file": base[:5],
        "no_length": base[:10],
        "hlen_zero": b"RDKVC001" + struct.pack("<I", 0) + base[12:],
        "hlen_huge": b"RDKVC001" + struct.pack("<I", (1 << 20) + 1) + base[12:],
        "header_truncated": base[:12 + hlen - 3],
        "bad_json": with_header("{\"L\":2,"),
        "json_trailing": with_header(htext + " x"),
        "not_object": with_header("[1,2]"),
        "missing_T": edit(T=None),
        "string_L": edit(L="2"),
        "dtype_f16": edit(dtype="f16"),
        "dtype_missing": edit(dtype=None),
        "q_not_multiple": edit(H_q=3),
        "zero_layers": edit(L=0),
        "sw_too_large": edit(S_w=17),
        "sw_zero": edit(S_w=0),
        "payload_truncated": base[:-4],
        "payload_trailing": base + b"\0",
        "nan_in_v": with_header(htext, bytes(nan_pl)),
        "inf_in_q": with_header(htext, bytes(inf_pl)),
        "fp16_overflow": with_header(htext, bytes(big_pl)),
    }
    out = {"names": np.array(list(variants))}
    for i, (name, data) in enumerate(variants.items()):
        p = os.path.join(tmp, f"v{i}.rdkvc")
        open(p, "wb").write(data)
        code, dims = ref.load_cache_status(p)
        out[f"bytes_{name}"] = np.frombuffer(data, np.uint8)
        out[f"status_{name}"] = np.int32(code)
        out[f"dims_{name}"] = dims
    np.savez_compressed(os.path.join(HERE, "cache_io.npz"), **out)


CALIB_CASES = [
    # (name, seeds, (L, Hq, Hkv, d, T), S_w, outliers, scale, widths, edit)
    ("basic", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], None),
    ("two_caches", [1, 2], (2, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], None),
    ("outliers", [7], (1, 2, 2, 32, 128), 32, 3, 100.0, [0, 2, 4, 8, 16], None),
    ("zero_units", [4], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], "zero_some"),
    ("widths_0_4_16", [5], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 4, 16], None),
    ("widths_0_16", [5], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 16], None),
    ("widths_2_8", [6], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 8, 16], None),
    ("fp16_values", [8], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], "fp16"),
    ("all_zero", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], "zero_all"),
    ("non_finite", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], "nan"),
    ("constant_units", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 2, 4, 8, 16], "const"),
    ("bad_widths", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0, 3, 16], None),
]


def make_calib():
    """calibrate_epsilon (quantizer.cpp:200-284) on the reference, both granularities."""
    out = {"names": np.array([c[0] for c in CALIB_CASES])}
    for name, seeds, (L, Hq, Hkv, d, T), sw, oc, osc, widths, ed in CALIB_CASES:
        ks, vs, qs = [], [], []
        for s in seeds:
            k, v, q = ref.gen_synthetic(s, L, Hq, Hkv, d, T, sw, oc, osc)
            ks.append(k), vs.append(v), qs.append(q)
        k, v, q = np.stack(ks), np.stack(vs), np.stack(qs)
        if ed == "zero_some":
            v[0, 0, 0, 3:9] = 0.0
            v[0, 0, 1, 60] = 0.0
            k[0, 0, 1, :, 5] = 0.0
            k[0, 0, 0, :, 0] = 0.0
        elif ed == "fp16":
            k, v = k.astype(np.float16).astype(np.float32), v.astype(np.float16).astype(np.float32)
        elif ed == "zero_all":
            k[:] = 0.0
            v[:] = 0.0
        elif ed == "nan":
            k[0, 0, 1, 7, 3] = np.nan
            v[0, 0, 0, 9, 2] = np.inf
        elif ed == "const":
            k[:] = 1.5
            v[:] = -0.25
        out[f"k_{name}"], out[f"v_{name}"] = k, v
        out[f"widths_{name}"] = np.array(widths, np.int32)
        for gran in (0, 1):
            try:
                eps, units = ref.calibrate(k, v, q, gran, widths)
                st = 0
            except RuntimeError as e:  # OracleError
                eps, units, st = np.zeros(len(widths)), 0, e.code
            out[f"eps_{name}_{gran}"] = eps
            out[f"units_{name}_{gran}"] = np.int64(units)
            out[f"status_{name}_{gran}"] = np.int32(st)
    np.savez_compressed(os.path.join(HERE, "calib.npz"), **out)


SWEEP_CASES = [
    # (name, seeds, (L, Hq, Hkv, d, T), S_w, outliers, scale, grid, cfg kwargs)
    ("basic", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0.25, 0.5, 1.0, 2.0, 4.0, 8.0, 16.0], {}),
    ("two_caches", [2, 3], (2, 4, 2, 16, 64), 16, 0, 1.0, [2.0, 0.5, 1.0], {}),
    ("outliers_window", [7], (1, 2, 2, 32, 128), 32, 3, 100.0, [1.0, 3.0], dict(window=8, pool_kernel=3)),
    ("widths_0_4_16", [5], (1, 4, 2, 16, 64), 16, 0, 1.0, [0.5, 2.0, 6.0], dict(widths=(0, 4, 16))),
    ("bad_grid_zero", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [0.0], {}),
    ("bad_grid_big", [1], (1, 4, 2, 16, 64), 16, 0, 1.0, [1.0, 17.0], {}),
]


def make_sweep():
    """run_sweep (sweep.cpp:40-114) + dual_bound (allocator.cpp:218-246) on the reference."""
    from paper_2605_08317_b200.pipeline import default_config
    out = {"names": np.array([c[0] for c in SWEEP_CASES])}
    for name, seeds, (L, Hq, Hkv, d, T), sw, oc, osc, grid, kw in SWEEP_CASES:
        ks, vs, qs = [], [], []
        for s in seeds:
            k, v, q = ref.gen_synthetic(s, L, Hq, Hkv, d, T, sw, oc, osc)
            ks.append(k), vs.append(v), qs.append(q)
        k, v, q = np.stack(ks), np.stack(vs), np.stack(qs)
        cfg = default_config(**kw)
        try:
            rows, st = ref.run_sweep(k, v, q, grid, cfg), 0
        except RuntimeError as e:  # OracleError
            rows, st = np.zeros((0, 5)), e.code
        out[f"k_{name}"], out[f"v_{name}"], out[f"q_{name}"] = k, v, q
        out[f"grid_{name}"] = np.array(grid, np.float64)
        out[f"cfg_{name}"] = np.frombuffer(bytes(cfg), np.uint8)
        out[f"rows_{name}"] = rows
        out[f"status_{name}"] = np.int32(st)
    np.savez_compressed(os.path.join(HERE, "sweep.npz"), **out)


def make_c1():
    """BASELINE configs[0]: 1 layer, 32 q / 8 kv heads, d=128, T=4096, n=128."""
    L, Hq, Hkv, d, T, Sw = 1, 32, 8, 128, 4096, 32
    k, v, pq = ref.gen_synthetic(1, L, Hq, Hkv, d, T, Sw)
    cfg = oracle.default_config()
    model = oracle.RefModel(ref, k, v, pq, cfg)
    q = orc.normal_stream(2024, L * Hq * d).reshape(L, Hq, d)
    outd, _ = model.decode(q)
    out = {"sha_k": np.frombuffer(hashlib.sha256(k.tobytes()).digest(), np.uint8),
           "sha_v": np.frombuffer(hashlib.sha256(v.tobytes()).digest(), np.uint8),
           "sha_q": np.frombuffer(hashlib.sha256(pq.tobytes()).digest(), np.uint8),
           "q": q, "out": outd}
    for h in range(Hkv):
        r = model.head(0, h)
        for key in ("v_bits", "k_bits"):
            out[f"h{h}_{key}"] = r[key].astype(np.uint8)
        for key in ("v_weights", "k_weights"):
            out[f"h{h}_{key}"] = r[key]
        for key in ("lambda_v", "lambda_k", "objective_v", "objective_k", "achieved_bits",
                    "v_converged", "k_converged", "n_kept"):
            out[f"h{h}_{key}"] = np.asarray(r[key])
        c = model.trizone(0, h).canon()
        out[f"h{h}_payload"] = c["payload"]
        out[f"h{h}_kept"] = c["kept"]
        out[f"h{h}_vscale"] = c["vscale"]
        out[f"h{h}_vzero"] = c["vzero"]
        out[f"h{h}_kscale"] = c["kscale"]
        out[f"h{h}_kzero"] = c["kzero"]
        out[f"h{h}_segtab"] = c["segtab"]
        out[f"h{h}_perm"] = c["perm"]
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)


if __name__ == "__main__":
    make_gen()
    make_alloc()
    make_trizone()
    make_mckp()
    make_c1()
    make_cache_io()
    make_calib()
    make_sweep()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
