"""Parity at the BASELINE.json shapes the bench runs (VERDICT r1 "untested
configurations"), on the same K0 inputs the bench generates:

  * configs[2]: one (sequence, layer) slice of the 128K LLaMA-3.1-8B workload
    against the UNMODIFIED reference (oracle/_ref: allocate_model +
    build_packed_model + packed_decode_step, trizone.cpp:91-305) — allocation,
    zone indices and payload bytes bit-exact, decode <= 1e-3 through the fp16
    production decode;
  * configs[3]: Qwen2.5-7B (g=7) / Mistral-7B (g=4) KV shapes at budgets whose
    mixed 2/4/8-bit tiles do not fit shared memory, decoded through the
    automatic dispatch and checked against the oracle's TriZone decode;
  * configs[4]: the LLaMA-3.1-70B KV shape (80 layers, GQA group 8) in one
    launch against the oracle, allocation of a layer against the reference.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, gen_chunk

pytestmark = pytest.mark.gpu

DECODE_TOL = 1e-3


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _slice(spec, b=0, layer=0):
    """Device K0 chunk of one (sequence, layer) and its host f32 copy (FP16-representable)."""
    k, v, q = gen_chunk(spec, b, layer)
    return (k, v, q), (k.float().cpu().numpy(), v.float().cpu().numpy(), q.float().cpu().numpy())


def test_configs2_128k_slice_matches_reference(cuda, ref):
    """Sequence 0, layer 0 of the bench workload (8 KV heads x 32 q-heads, T=131072, n=128)."""
    spec = WorkloadSpec(batch=1, layers=1, ctx=131072, n_tokens=128)
    (kd, vd, qd), (k, v, q) = _slice(spec)
    H, T, d, g, Sw = spec.kv_heads, spec.ctx, spec.head_dim, spec.group, spec.probe_rows
    cfg = P.default_config(n_tokens=spec.n_tokens, window=Sw)
    al = P.allocate_model(kd, qd, cfg, kv_heads=H)
    al.check()
    model = P.build_packed_model(kd, vd, al, group=g)
    model.check()
    rm = oracle.RefModel(ref, k[None], v[None], q.reshape(1, H * g, Sw, d), oracle.default_config(n_tokens=128, window=Sw))
    vb, kb, st = al.v_bits.cpu().numpy(), al.k_bits.cpu().numpy(), al.stats_host()
    for h in range(H):
        want = rm.head(0, h)
        assert np.array_equal(vb[h], want["v_bits"]), h
        assert np.array_equal(kb[h][: len(want["k_bits"])], want["k_bits"]), h
        # the integer allocation is bit-exact end to end; lambda and the objectives are
        # fp64 functions of the weights, which differ from the reference's by a few ulps
        # (fp64 tensor-core probe dots in another association): a tight relative bound
        assert st[h]["achieved_bits"] == want["achieved_bits"], h
        for f in ("lambda_v", "lambda_k", "objective_v", "objective_k"):
            assert abs(st[h][f] - want[f]) <= 1e-4 * abs(want[f]), (h, f, st[h][f], want[f])
        got, exp = model.export(h), rm.trizone(0, h).canon()
        for f in ("kept", "payload", "segtab", "perm", "vscale", "vzero", "kscale", "kzero"):
            assert np.array_equal(got[f], exp[f]), (h, f)
    assert model.plan.uniform2 >= 1  # the production (u2x) kernel decodes this slice
    qn = oracle.load().normal_stream(0xD15C0, H * g * d).reshape(H, g, d).astype(np.float16).astype(np.float32)
    out = P.packed_decode_step(model, torch.from_numpy(qn).to(cuda).half()).float().cpu().numpy()
    want, _ = rm.decode(qn.reshape(1, H * g, d))
    worst = max(rel(out.reshape(H * g, d)[j], want[0, j]) for j in range(H * g))
    assert worst < DECODE_TOL, worst


@pytest.mark.parametrize("name,Hq,Hkv,n", [("qwen2.5-7b", 28, 4, 1024), ("qwen2.5-7b", 28, 4, 2048),
                                           ("mistral-7b", 32, 8, 2048), ("qwen2.5-7b", 28, 4, 256),
                                           ("mistral-7b", 32, 8, 64)])
def test_configs3_large_mixed_tiles_auto_dispatch(cuda, orc, name, Hq, Hkv, n):
    """configs[3] budget points (64 .. 3,100 kept slots at mixed 2/4 bits, heavy hitters
    + outlier K channels, the bench's inputs): the automatic dispatch (the chunked
    split-K mixed 2/4-bit kernel, decode_u24) vs the oracle's build_trizone +
    packed_decode_step; the same step without split-K (no partials workspace, one
    warp pair per tile) and with f32 I/O must agree too."""
    spec = WorkloadSpec(batch=1, layers=2, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                        hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
    g, d = spec.group, spec.head_dim
    cfg = P.default_config(n_tokens=n, window=spec.probe_rows)
    rng = np.random.default_rng(n + Hq)
    worst, classes = 0.0, set()
    for layer in range(spec.layers):
        (kd, vd, qd), (k, v, _) = _slice(spec, 0, layer)
        al = P.allocate_model(kd, qd, cfg, kv_heads=Hkv)
        al.check()
        model = P.build_packed_model(kd, vd, al, group=g)
        model.check()
        if n >= 1024:
            assert model.plan.max_slots > 1024
        assert model.plan.mix24
        q = rng.standard_normal((Hkv, g, d)).astype(np.float16).astype(np.float32)
        out = P.packed_decode_step(model, torch.from_numpy(q).to(cuda).half()).float().cpu().numpy()
        ws, model.split_ws = model.split_ws, None  # one pair per tile, no partials
        out1 = P.packed_decode_step(model, torch.from_numpy(q).to(cuda)).cpu().numpy()
        model.split_ws = ws
        assert rel(out1, out) < 1e-3
        vb, kb = al.v_bits.cpu().numpy(), al.k_bits.cpu().numpy()
        for h in range(Hkv):
            classes |= set(np.unique(vb[h]).tolist())
            tz = orc.tz_build(k[h], v[h], vb[h].astype(np.int32), kb[h].astype(np.int32))
            for j in range(g):
                worst = max(worst, rel(out[h, j], tz.decode(q[h, j])))
    assert {2, 4}.issubset(classes), classes  # mixed tiers, not the uniform fast path
    assert worst < DECODE_TOL, worst


@pytest.mark.parametrize("name,L,Hq,Hkv,n", [("mistral-7b", 32, 32, 8, 256), ("qwen2.5-7b", 28, 28, 4, 1024)])
def test_configs3_full_step_split_k(cuda, name, L, Hq, Hkv, n):
    """A whole configs[3] step (batch 4, every layer: 448 / 1024 tiles) has more
    (tile, part) items than warp pairs, so the chunked split-K kernel deals items
    over several rounds and merges the parts. The step must equal the
    one-pair-per-tile decode (no partials) and the CUDA-core kernel, and repeat
    bit-identically."""
    from paper_2605_08317_b200.workload import build

    spec = WorkloadSpec(batch=4, layers=L, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                        hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
    m, _, _, _ = build(spec)
    assert m.plan.mix24 and m.split_ws is not None
    q = P.generate((m.units, spec.group, spec.head_dim), torch.float16, seed=5, tensor=2)
    a = P.packed_decode_step(m, q)
    outs = [P.packed_decode_step(m, q) for _ in range(3)]
    for o in outs:
        assert torch.equal(o, a)
    gen = P.packed_decode_step(m, q, kernel=1).float()
    ws, m.split_ws = m.split_ws, None
    whole = P.packed_decode_step(m, q).float()
    m.split_ws = ws
    assert rel(a.float().cpu(), gen.cpu()) < DECODE_TOL
    assert rel(whole.cpu(), a.float().cpu()) < DECODE_TOL


def test_configs4_llama70b_g8_all_layers(cuda, orc, ref):
    """configs[4] LLaMA-3.1-70B KV shape: 80 layers x 8 KV heads, GQA group 8, n=128,
    in one decode launch (two 4-head passes per staged tile). T reduced to 8K so the
    oracle can decode all 640 tiles; the tile shapes match 128K (128 kept tokens, 2 bits)."""
    spec = WorkloadSpec(batch=1, layers=80, q_heads=64, kv_heads=8, ctx=8192, n_tokens=128, seed=5)
    H, g, d, Sw = spec.kv_heads, spec.group, spec.head_dim, spec.probe_rows
    cfg = P.default_config(n_tokens=128, window=Sw)
    Ks, Vs, vbs, kbs = [], [], [], []
    host = []
    checked = (0, 1, 39, 79)  # layers decoded by the oracle (all 80 run in the launch)
    for layer in range(spec.layers):
        k, v, qp = gen_chunk(spec, 0, layer)
        al = P.allocate_model(k, qp, cfg, kv_heads=H)
        al.check()
        Ks.append(k), Vs.append(v), vbs.append(al.v_bits), kbs.append(al.k_bits)
        if layer in checked:
            hk = (k.float().cpu().numpy(), v.float().cpu().numpy(),
                  qp.float().cpu().numpy() if layer == 0 else None)
            host.append((layer, hk, al))
    K, V = torch.cat(Ks), torch.cat(Vs)
    alloc = P.Allocation(torch.cat(vbs), torch.cat(kbs), torch.zeros(1, dtype=torch.uint8, device=cuda))
    model = P.build_packed_model(K, V, alloc, group=g)
    model.check()
    assert model.units == 640 and model.plan.uniform2 >= 1
    rng = np.random.default_rng(70)
    q = rng.standard_normal((640, g, d)).astype(np.float16).astype(np.float32)
    out = P.packed_decode_step(model, torch.from_numpy(q).to(cuda).half()).float().cpu().numpy()
    worst = 0.0
    for layer, (k, v, pq), al in host:
        vb, kb = al.v_bits.cpu().numpy(), al.k_bits.cpu().numpy()
        if pq is not None:  # allocation of this layer vs the reference
            rm = oracle.RefModel(ref, k[None], v[None], pq.reshape(1, H * g, Sw, d), oracle.default_config(n_tokens=128, window=Sw))
            for h in range(H):
                want = rm.head(0, h)
                assert np.array_equal(vb[h], want["v_bits"]) and np.array_equal(kb[h][: len(want["k_bits"])], want["k_bits"])
        for h in range(H):
            u = layer * H + h
            tz = orc.tz_build(k[h], v[h], vb[h].astype(np.int32), kb[h].astype(np.int32))
            for j in range(g):
                worst = max(worst, rel(out[u, j], tz.decode(q[u, j])))
    assert worst < DECODE_TOL, worst


@pytest.mark.parametrize("T,strict,force", [(8192, False, False), (40000, True, False), (131072, False, True)])
def test_long_context_allocation_given_weights(cuda, orc, T, strict, force):
    """Long contexts take the cluster-parallel V sweep (allocate.cu allocate_v_cluster,
    T >= 8192) and allocate_finish: v_bits / k_bits / lambdas / convergence /
    objectives bit-identical to the C restatement of mckp_bisect (allocator.cpp:135-216)
    on the same f32 weights, for flat, peaky and heavy-hitter weight shapes."""
    rng = np.random.default_rng(T)
    d, Hkv, n = 128, 8, 128
    flat = rng.random(T).astype(np.float32) * 1e-4
    peaky = (rng.standard_exponential(T) ** 4).astype(np.float32) * 1e-6
    heavy = flat.copy()
    heavy[::64] *= 300.0
    w_t = np.stack([flat, peaky, heavy])
    w_c = (rng.random((3, d)) * np.linspace(0.5, 4.0, d)).astype(np.float32)
    cfg = oracle.default_config(n_tokens=n, window=32, strict_budget=strict, force_window_retain=force)
    al = P.allocate(torch.from_numpy(w_t).to(cuda), torch.from_numpy(w_c).to(cuda), P.default_config(
        n_tokens=n, window=32, strict_budget=strict, force_window_retain=force), group=4, probe_rows=32, kv_heads=Hkv)
    al.check()
    st, vb, kb = al.stats_host(), al.v_bits.cpu().numpy(), al.k_bits.cpu().numpy()
    bud = orc.head_budget(n, 0.5, d, Hkv)
    widths = [cfg.widths[i] for i in range(cfg.n_widths)]
    eps_v = [cfg.eps_v[i] for i in range(cfg.n_widths)]
    eps_k = [cfg.eps_k[i] for i in range(cfg.n_widths)]
    for u in range(3):
        want = orc.mckp_bisect(w_t[u], widths, eps_v, min(16.0, bud["v_bits"] / (d * T)), strict_budget=strict)
        wb = want["bits"].copy()
        if force:
            wb[T - 32:] = 16
        assert np.array_equal(vb[u], wb), u
        assert st[u]["lambda_v"] == want["lambda"] and bool(st[u]["v_converged"]) == want["converged"], u
        kept = int(np.count_nonzero(wb))
        assert st[u]["n_kept"] == kept
        if not force:
            assert st[u]["objective_v"] == want["objective"], u
        wk = orc.mckp_bisect(w_c[u], widths, eps_k, min(16.0, bud["k_bits"] / (kept * d)), strict_budget=strict)
        assert np.array_equal(kb[u], wk["bits"]) and st[u]["lambda_k"] == wk["lambda"], u
        assert st[u]["objective_k"] == wk["objective"], u


def test_streaming_weights_match_reference_long(cuda, ref):
    """Stage-1 weights at T=16384 through the streaming two-pass K1 (no probe matrix in
    HBM) vs the reference's attention_probe + token_weights + channel_weights:
    <= 1e-6 relative, and nearly all f32 values bit-identical."""
    spec = WorkloadSpec(batch=1, layers=1, ctx=16384, n_tokens=128, seed=3, hh_stride=64, hh_boost=1.0)
    (kd, vd, qd), (k, v, q) = _slice(spec)
    H, g, d, Sw = spec.kv_heads, spec.group, spec.head_dim, spec.probe_rows
    w_t, w_c = P.compute_weights(kd[:2], qd[:2], window=Sw, pool_kernel=5, kv_heads=H)
    w_t, w_c = w_t.cpu().numpy(), w_c.cpu().numpy()
    rm = oracle.RefModel(ref, k[None], v[None], q.reshape(1, H * g, Sw, d), oracle.default_config(n_tokens=128, window=Sw))
    exact = total = 0
    for h in range(2):
        want = rm.head(0, h)
        for got, exp in ((w_t[h], want["v_weights"]), (w_c[h], want["k_weights"])):
            assert np.max(np.abs(got - exp) / np.maximum(np.abs(exp), 1e-30)) <= 1e-6
            exact += int(np.sum(got == exp))
            total += got.size
    assert exact / total > 0.99, exact / total


def test_weights_unit_boundaries_bit_identical(cuda):
    """The persistent probe kernel walks (unit, token tile) ranges that cross units
    inside a CTA (the unit's probe rows are swapped in shared memory there): the
    weights of every unit must equal those of the unit computed alone, bit for bit,
    and two runs must agree."""
    spec = WorkloadSpec(batch=1, layers=1, ctx=12288, n_tokens=128, seed=9, hh_stride=64, hh_boost=1.0)
    (kd, vd, qd), _ = _slice(spec)
    H, Sw = spec.kv_heads, spec.probe_rows
    w_t, w_c = P.compute_weights(kd, qd, window=Sw, pool_kernel=5, kv_heads=H)
    w_t2, w_c2 = P.compute_weights(kd, qd, window=Sw, pool_kernel=5, kv_heads=H)
    assert torch.equal(w_t, w_t2) and torch.equal(w_c, w_c2)
    for h in range(H):
        a_t, a_c = P.compute_weights(kd[h:h + 1].contiguous(), qd[h:h + 1].contiguous(), window=Sw, pool_kernel=5,
                                     kv_heads=H)
        assert torch.equal(a_t[0], w_t[h]) and torch.equal(a_c[0], w_c[h]), h


def test_weights_logit_batches_bit_identical(cuda):
    """S1 stores the logits of at most 2 GiB of units at a time (R x T fp64 per
    unit) and S3 reads them back: 9 units of T = 262144 (268 MB each) run as two
    batches, and every unit must equal the unit computed alone."""
    g_, rows, T, U = 4, 32, 262144, 9
    gen = torch.Generator(device="cuda").manual_seed(21)
    k = (torch.randn((U, T, 128), generator=gen, device="cuda") * 0.5).half()
    q = (torch.randn((U, g_, rows, 128), generator=gen, device="cuda") * 0.5).half()
    w_t, w_c = P.compute_weights(k, q, window=rows, pool_kernel=5, kv_heads=U)
    assert torch.isfinite(w_t).all() and float(w_t.sum()) > 0
    for u in (0, 7, 8):  # first batch, its last unit, the second batch
        a_t, a_c = P.compute_weights(k[u:u + 1].contiguous(), q[u:u + 1].contiguous(), window=rows, pool_kernel=5,
                                     kv_heads=U)
        assert torch.equal(a_t[0], w_t[u]) and torch.equal(a_c[0], w_c[u]), u
