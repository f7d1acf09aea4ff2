"""Tensor-core decode kernel (csrc/decode_mma.cu) vs the oracle and vs the generic kernel.

Covers every bit class of V rows and K channels, Zone B (16-bit V rows),
k16 (16-bit K channels), Zone C appends, GQA groups 1..8, fp16 and f32 I/O,
and batches of many tiles in one persistent launch.
"""
import numpy as np
import pytest
import torch

from paper_2605_08317_b200 import capi
from paper_2605_08317_b200 import pipeline as P

pytestmark = pytest.mark.gpu

D = 128
FP16_INPUT_TOL = 1e-4
# uniform-2-bit fast path (csrc/decode_mma.cu u2x): 16-bit softmax weights,
# typically 1e-5 .. 3e-4 relative on random data, worst seen 5.4e-4; the
# contract is 1e-3 (DECODE_TOL in test_gpu_parity.py)
U2X_TOL = 1e-3


def f16r(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def _random_case(rng, T, g, p_bits=(0.2, 0.2, 0.2, 0.2, 0.2), kp=(0.2, 0.2, 0.2, 0.2, 0.2), max16=60):
    choices = np.array([0, 2, 4, 8, 16])
    k = f16r(rng.standard_normal((T, D)) * rng.uniform(0.3, 3.0))
    v = f16r(rng.standard_normal((T, D)))
    vb = choices[rng.choice(5, T, p=p_bits)].astype(np.int32)
    idx16 = np.nonzero(vb == 16)[0]
    if len(idx16) > max16:
        vb[idx16[max16:]] = 8
    vb[rng.integers(0, T)] = 2
    kb = choices[rng.choice(5, D, p=kp)].astype(np.int32)
    q = f16r(rng.standard_normal((g, D)))
    return k, v, vb, kb, q


def _run_batch(cuda, orc, cases, g, io=torch.float32, appends=0, rng=None, tol=FP16_INPUT_TOL):
    """Pack all cases (same T) as units of one model; decode with both kernels."""
    T = cases[0][0].shape[0]
    K = torch.from_numpy(np.stack([c[0] for c in cases])).to(cuda)
    V = torch.from_numpy(np.stack([c[1] for c in cases])).to(cuda)
    vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).to(cuda)
    kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).to(cuda)
    stats = torch.zeros(len(cases) * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device=cuda)
    model = P.build_packed_model(K, V, P.Allocation(vb, kb, stats), group=g, zc_cap=appends)
    model.check()
    zk = zv = None
    if appends:
        zk = f16r(rng.standard_normal((appends, len(cases), D)))
        zv = f16r(rng.standard_normal((appends, len(cases), D)))
        for a in range(appends):
            P.append_new_token(model, torch.from_numpy(zk[a]).to(cuda), torch.from_numpy(zv[a]).to(cuda))
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).to(io)
    out_mma = P.packed_decode_step(model, q, kernel=2).float().cpu().numpy()
    out_gen = P.packed_decode_step(model, q, kernel=1).float().cpu().numpy()
    worst = 0.0
    for u, (k, v, vbs, kbs, qq) in enumerate(cases):
        tz = orc.tz_build(k, v, vbs, kbs)
        for a in range(appends):
            tz.append(zk[a, u], zv[a, u])
        for j in range(g):
            want = tz.decode(qq[j])
            worst = max(worst, rel(out_mma[u, j], want))
            assert rel(out_mma[u, j], out_gen[u, j]) < (2 * tol if io == torch.float32 else 1e-3)
    return worst, model


def test_mma_all_two_bit_default_budget_shape(cuda, orc):
    """The C1/C3 allocation shape: 128 kept tokens, every V row and K channel at 2 bits."""
    rng = np.random.default_rng(1)
    cases = []
    for _ in range(16):
        k, v, vb, kb, q = _random_case(rng, 512, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(512, 128, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, 4, tol=U2X_TOL)
    assert model.plan.max_slots == 128 and model.plan.uniform2 == 2  # uniform 2-bit, all K channels kept
    assert worst < U2X_TOL, worst
    # the specialised uniform-2-bit body and the general tensor-core body agree
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda)
    a = P.packed_decode_step(model, q, kernel=2)
    for k in (3, 4):  # general body, one-warp uniform body (kernel 2 = warp-pair body)
        b = P.packed_decode_step(model, q, kernel=k)
        assert float(((a - b).norm(dim=-1) / b.norm(dim=-1)).max()) < 2 * U2X_TOL, k


@pytest.mark.parametrize("g", [1, 2, 4, 7, 8])
def test_mma_mixed_classes(cuda, orc, g):
    rng = np.random.default_rng(100 + g)
    cases = [_random_case(rng, 280, g) for _ in range(12)]
    worst, model = _run_batch(cuda, orc, cases, g)
    assert model.plan.max_slots <= 256
    assert worst < FP16_INPUT_TOL, worst


@pytest.mark.parametrize("g", [4, 7])
def test_mma_long_mixed_tiles(cuda, orc, g):
    """Mixed-bit tiles well past 256 slots (configs[3] budgets n >= 256) stay on the
    tensor-core general body while the whole tile fits in shared memory."""
    rng = np.random.default_rng(500 + g)
    T = 900 if g <= 4 else 540  # g > 4 runs two 4-head passes with twice the scratch
    cases = [_random_case(rng, T, g, p_bits=(0.15, 0.35, 0.3, 0.15, 0.05)) for _ in range(6)]
    worst, model = _run_batch(cuda, orc, cases, g)
    assert model.plan.max_slots > 400 and model.plan.uniform2 == 0
    assert worst < FP16_INPUT_TOL, worst


def test_mma_tile_too_big_for_smem_falls_back(cuda):
    """A tile whose packed bytes exceed shared memory: automatic dispatch runs the
    CUDA-core kernel, forcing the tensor-core path is an invalid argument."""
    rng = np.random.default_rng(9)
    cases = [_random_case(rng, 3000, 4, p_bits=(0.05, 0.05, 0.1, 0.8, 0.0)) for _ in range(2)]
    K = torch.from_numpy(np.stack([c[0] for c in cases])).to(cuda)
    V = torch.from_numpy(np.stack([c[1] for c in cases])).to(cuda)
    vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).to(cuda)
    kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).to(cuda)
    stats = torch.zeros(len(cases) * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device=cuda)
    model = P.build_packed_model(K, V, P.Allocation(vb, kb, stats), group=4)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda)
    a = P.packed_decode_step(model, q)
    b = P.packed_decode_step(model, q, kernel=1)
    assert torch.equal(a, b)
    with pytest.raises(capi.InvalidArgument):
        P.packed_decode_step(model, q, kernel=2)


def test_mma_zone_c_and_fp16_io(cuda, orc):
    rng = np.random.default_rng(7)
    cases = [_random_case(rng, 200, 4) for _ in range(9)]
    worst, _ = _run_batch(cuda, orc, cases, 4, appends=6, rng=rng)
    assert worst < FP16_INPUT_TOL, worst
    worst, _ = _run_batch(cuda, orc, cases, 4, io=torch.float16, appends=3, rng=rng)
    assert worst < 1e-3, worst


def test_mma_edge_allocations(cuda, orc):
    rng = np.random.default_rng(9)
    T = 64
    base = _random_case(rng, T, 4)
    cases = []
    # all K channels removed -> uniform attention over V_hat
    k, v, vb, kb, q = [x.copy() for x in base]
    kb[:] = 0
    cases.append((k, v, vb, kb, q))
    # all K channels 16-bit (k16 only)
    k, v, vb, kb, q = [x.copy() for x in base]
    kb[:] = 16
    cases.append((k, v, vb, kb, q))
    # single kept token at 8 bits
    k, v, vb, kb, q = [x.copy() for x in base]
    vb[:] = 0
    vb[5] = 8
    cases.append((k, v, vb, kb, q))
    # constant V row and constant K column (degenerate 1e-12 ranges)
    k, v, vb, kb, q = [x.copy() for x in base]
    v[:, :] = f16r(1.25)
    k[:, 3] = f16r(-0.5)
    cases.append((k, v, vb, kb, q))
    worst, _ = _run_batch(cuda, orc, cases, 4)
    assert worst < FP16_INPUT_TOL, worst


def test_mma_large_batch_persistent(cuda, orc):
    """More tiles than resident warps: every worker walks several tiles through its ring."""
    rng = np.random.default_rng(11)
    cases = []
    for i in range(600):
        k, v, vb, kb, q = _random_case(rng, 96, 4, p_bits=(0.4, 0.3, 0.15, 0.1, 0.05))
        cases.append((k, v, vb, kb, q))
    # check only a sample against the oracle (all against the generic kernel)
    worst, _ = _run_batch(cuda, orc, cases[:40], 4)
    assert worst < FP16_INPUT_TOL
    T = 96
    K = torch.from_numpy(np.stack([c[0] for c in cases])).to(cuda)
    V = torch.from_numpy(np.stack([c[1] for c in cases])).to(cuda)
    vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).to(cuda)
    kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).to(cuda)
    stats = torch.zeros(len(cases) * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device=cuda)
    model = P.build_packed_model(K, V, P.Allocation(vb, kb, stats), group=4)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda)
    a = P.packed_decode_step(model, q, kernel=2)
    b = P.packed_decode_step(model, q, kernel=1)
    err = (a - b).norm(dim=-1) / b.norm(dim=-1)
    assert float(err.max()) < 2 * FP16_INPUT_TOL
    del T


@pytest.mark.parametrize("g,fullk,io", [(4, True, torch.float32), (4, True, torch.float16), (4, False, torch.float32),
                                        (1, True, torch.float32), (2, False, torch.float16), (3, True, torch.float32),
                                        (8, True, torch.float16), (7, False, torch.float32), (5, True, torch.float32)])
def test_mma_uniform_two_bit_ragged(cuda, orc, g, fullk, io):
    """Uniform 2-bit tiles of every block count (1..160 kept tokens, ragged last
    block), with all K channels kept (identity channel_perm) or some dropped;
    GQA groups of 5..8 heads run as two 4-head passes over each staged tile."""
    rng = np.random.default_rng(40 + g + 10 * fullk)
    cases = []
    for n in (1, 3, 31, 32, 33, 64, 65, 100, 127, 128, 129, 131, 150, 157, 160):
        k, v, vb, kb, q = _random_case(rng, 400, g)
        vb[:] = 0
        vb[np.sort(rng.choice(400, n, replace=False))] = 2
        kb[:] = 2
        if not fullk:
            kb[rng.choice(D, 9, replace=False)] = 0
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, g, io=io, tol=U2X_TOL)
    assert model.plan.uniform2 == (2 if fullk else 1)
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_pipelined_host_decode_matches_device(cuda, orc, chunks):
    """rdkv_cuda_decode_host_pipelined (chunked H2D / decode / D2H overlap) returns
    exactly the device-path outputs, for chunk counts that do not divide the units."""
    rng = np.random.default_rng(5 + chunks)
    cases = []
    for _ in range(37):
        k, v, vb, kb, q = _random_case(rng, 300, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(300, int(rng.integers(90, 160)), replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    _, model = _run_batch(cuda, orc, cases, 4, tol=U2X_TOL)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).half()
    want = P.packed_decode_step(model, q).cpu()
    dec = P.HostDecoder(model, torch.float16, chunks=chunks)
    qh = q.cpu().pin_memory()
    oh = torch.full_like(qh, float("nan")).pin_memory()
    for _ in range(2):  # reuse of the context and staging buffers
        dec.step(qh, oh)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(oh, want)
    dec.close()


@pytest.mark.parametrize("io", [torch.float16, torch.float32])
def test_host_decode_zero_copy_and_pageable(cuda, orc, io):
    """rdkv_cuda_decode_host: pinned buffers go zero-copy (the kernel streams q
    in and out over PCIe), pageable ones through the staging copies; both equal
    the device path bit for bit."""
    import ctypes as C

    rng = np.random.default_rng(77)
    cases = []
    for _ in range(21):
        k, v, vb, kb, q = _random_case(rng, 300, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(300, int(rng.integers(60, 160)), replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    _, model = _run_batch(cuda, orc, cases, 4, tol=U2X_TOL)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).to(io)
    want = P.packed_decode_step(model, q).cpu()
    qd, od = torch.empty_like(q), torch.empty_like(q)
    a = P.decode_args(model, qd, od)
    L = capi.lib()
    st = torch.cuda.current_stream().cuda_stream
    for pinned in (True, False):
        qh = q.cpu()
        oh = torch.full_like(qh, float("nan"))
        if pinned:
            qh, oh = qh.pin_memory(), oh.pin_memory()
        assert L.rdkv_cuda_decode_host(C.byref(a), qh.data_ptr(), oh.data_ptr(), st) == 0
        torch.cuda.synchronize()
        assert torch.equal(oh, want), pinned


@pytest.mark.parametrize("g,fullk,io", [(4, True, torch.float16), (4, False, torch.float32), (2, True, torch.float32)])
def test_mma_uniform_two_bit_long_tiles(cuda, orc, g, fullk, io):
    """Uniform 2-bit tiles longer than 160 slots (the configs[3] budget sweep):
    the chunked u2x kernel with an online softmax across <= 160-slot chunks,
    mixed with short tiles in the same launch."""
    rng = np.random.default_rng(60 + g + 10 * fullk)
    cases = []
    for n in (5, 128, 161, 200, 333, 512, 700, 1100):
        k, v, vb, kb, q = _random_case(rng, 1200, g)
        vb[:] = 0
        vb[np.sort(rng.choice(1200, n, replace=False))] = 2
        kb[:] = 2
        if not fullk:
            kb[rng.choice(D, 5, replace=False)] = 0
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, g, io=io, tol=U2X_TOL)
    assert model.plan.max_slots > 1000 and model.plan.uniform2 == (2 if fullk else 1)
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst


@pytest.mark.parametrize("n_max,appends,io", [(150, 1, torch.float16), (150, 17, torch.float32), (600, 40, torch.float16),
                                              (130, 5, torch.float32), (128, 3, torch.float32), (160, 4, torch.float16),
                                              (600, 2, torch.float32), (132, 9, torch.float16), (160, 16, torch.float32),
                                              (128, 12, torch.float16)])
def test_mma_uniform_two_bit_zone_c(cuda, orc, n_max, appends, io):
    """Zone C (appended fp16 K/V rows) on the uniform-2-bit fast path: up to 4
    (or, in the long-generation variant, 16) rows staged with each short tile
    (fused), more as 16-token fp16 tensor-core chunks folded into the online
    softmax, after short or chunked long packed tiles."""
    rng = np.random.default_rng(80 + appends)
    cases = []
    for n in (3, 64, 100, n_max):
        k, v, vb, kb, q = _random_case(rng, 700, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(700, n, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, 4, io=io, appends=appends, rng=rng, tol=U2X_TOL)
    assert model.plan.uniform2 == 2
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst


@pytest.mark.parametrize("appends,known", [(2, True), (6, True), (2, False)])
def test_host_decode_zero_copy_zone_c(cuda, orc, appends, known):
    """Zero-copy host decode (TMA bulk stores to mapped host memory) with Zone C
    rows: fused (host-known bound <= 4) and chunked paths equal the device path."""
    import ctypes as C

    rng = np.random.default_rng(90 + appends)
    cases = []
    for n in (2, 90, 128, 150):
        k, v, vb, kb, q = _random_case(rng, 400, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(400, n, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    _, model = _run_batch(cuda, orc, cases, 4, appends=appends, rng=rng, tol=U2X_TOL)
    if not known:
        model.zc_count = None
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).half()
    # the zero-copy path stages Zone C itself (fused / chunked): compare with the device
    # step on the same variant (no prepass workspace), and with the prepass step to 1e-3
    tiny = torch.empty(1, dtype=torch.uint8, device=cuda)
    want = P.packed_decode_step(model, q, workspace=tiny).cpu()
    pre = P.packed_decode_step(model, q).float().cpu()
    assert float(((pre - want.float()).norm() / want.float().norm()).item()) < 1e-3
    qd, od = torch.empty_like(q), torch.empty_like(q)
    a = P.decode_args(model, qd, od, workspace=tiny)
    qh = q.cpu().pin_memory()
    oh = torch.full_like(qh, float("nan")).pin_memory()
    assert capi.lib().rdkv_cuda_decode_host(C.byref(a), qh.data_ptr(), oh.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(oh, want)


@pytest.mark.parametrize("io,g", [(torch.float16, 4), (torch.float32, 4), (torch.float16, 8), (torch.float32, 6)])
def test_split_dispatch_mixed_arena(cuda, orc, io, g):
    """An arena of mostly uniform-2-bit tiles plus a few mixed ones (the heavy-
    hitter shape): the split step (mixed tiles on the general body, uniform ones
    on u2x through unit_ids) equals the all-general step and the oracle."""
    rng = np.random.default_rng(123)
    cases = []
    for i in range(40):
        k, v, vb, kb, q = _random_case(rng, 300, g)
        vb[:] = 0
        vb[np.sort(rng.choice(300, int(rng.integers(100, 150)), replace=False))] = 2
        kb[:] = 2
        if i % 7 == 3:  # 8-bit rows and a Zone B row (not 2/4/8-bit only: the general body)
            vb[np.nonzero(vb)[0][:3]] = 8
            vb[np.nonzero(vb)[0][3]] = 16
            kb[rng.choice(D, 3, replace=False)] = 4
        elif i % 7 == 5:  # a few 4-bit rows / channels (the MIX kernel)
            vb[np.nonzero(vb)[0][:3]] = 4
            kb[rng.choice(D, 3, replace=False)] = 4
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, g, io=io)
    plan = model.plan
    assert plan.uniform2 == 0 and 0 < plan.n_uniform < len(cases) and not plan.mix24
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).to(io)
    split = P.packed_decode_step(model, q)
    ids, model.unit_ids = model.unit_ids, None
    general = P.packed_decode_step(model, q)
    model.unit_ids = ids
    err = (split.float() - general.float()).norm(dim=-1) / general.float().norm(dim=-1)
    assert float(err.max()) < (2 * U2X_TOL if io == torch.float32 else 2e-3)


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_pipelined_host_decode_mixed_arena(cuda, orc, chunks):
    """The pipelined end-to-end call on a mixed arena that carries split lists
    (unit_ids): per-chunk launches drop the whole-arena ids (they would index
    past the chunk's shifted offsets / q / out), outputs equal the oracle and
    the no-split device step."""
    rng = np.random.default_rng(77 + chunks)
    cases = []
    for i in range(30):
        k, v, vb, kb, q = _random_case(rng, 300, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(300, int(rng.integers(100, 150)), replace=False))] = 2
        kb[:] = 2
        if i % 5 == 2:
            vb[np.nonzero(vb)[0][:3]] = 8
            kb[rng.choice(D, 3, replace=False)] = 4
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, 4, io=torch.float16)
    assert model.plan.uniform2 == 0 and 0 < model.plan.n_uniform < len(cases)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).half()
    ids, model.unit_ids = model.unit_ids, None
    want = P.packed_decode_step(model, q).cpu()
    model.unit_ids = ids
    dec = P.HostDecoder(model, torch.float16, chunks=chunks)
    qh = q.cpu().pin_memory()
    oh = torch.full_like(qh, float("nan")).pin_memory()
    dec.step(qh, oh)
    torch.cuda.current_stream().synchronize()
    dec.close()
    assert torch.equal(oh, want)
    for u, (k, v, vbs, kbs, qq) in enumerate(cases):
        tz = orc.tz_build(k, v, vbs, kbs)
        for j in range(4):
            assert rel(oh[u, j].float().numpy(), tz.decode(qq[j])) < 1e-3


def test_append_capacity_and_zone_c_bound(cuda, orc):
    """append_new_token past the Zone C capacity raises (no silently dropped
    rows); the HostDecoder's Zone C bound follows appends made after it was
    created (fused path for <= 4 rows, chunked beyond), matching the oracle."""
    rng = np.random.default_rng(9)
    cases = []
    for _ in range(12):
        k, v, vb, kb, q = _random_case(rng, 300, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(300, 120, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    cap = 7
    _, model = _run_batch(cuda, orc, cases, 4, io=torch.float16, appends=0)
    model.zc_k = torch.zeros((len(cases), cap, D), dtype=torch.float16, device=cuda)
    model.zc_v = torch.zeros_like(model.zc_k)
    model.zc_len = torch.zeros(len(cases), dtype=torch.int32, device=cuda)
    model.zc_cap, model.zc_count = cap, 0
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).half()
    dec = P.HostDecoder(model, torch.float16, chunks=2)
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    zk = f16r(rng.standard_normal((cap, len(cases), D)))
    zv = f16r(rng.standard_normal((cap, len(cases), D)))
    for a in range(cap):
        P.append_new_token(model, torch.from_numpy(zk[a]).to(cuda), torch.from_numpy(zv[a]).to(cuda))
        dec.step(qh, oh)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(oh, P.packed_decode_step(model, q).cpu())
        for u, (k, v, vbs, kbs, qq) in enumerate(cases):
            tz = orc.tz_build(k, v, vbs, kbs)
            for r in range(a + 1):
                tz.append(zk[r, u], zv[r, u])
            assert rel(oh[u, 0].float().numpy(), tz.decode(qq[0])) < 1e-3, (a, u)
    dec.close()
    with pytest.raises(capi.InvalidArgument):
        P.append_new_token(model, torch.from_numpy(zk[0]).to(cuda), torch.from_numpy(zv[0]).to(cuda))
    model.zc_count = None  # unknown bound: the capacity check reads zc_len on the device
    with pytest.raises(capi.InvalidArgument):
        P.append_new_token(model, torch.from_numpy(zk[0]).to(cuda), torch.from_numpy(zv[0]).to(cuda))


@pytest.mark.parametrize("world,appends,io", [(2, 0, torch.float16), (3, 0, torch.float32), (2, 20, torch.float32),
                                              (4, 3, torch.float16)])
def test_sequence_split_partials_merge(cuda, orc, world, appends, io):
    """Optional cross-GPU merge, simulated in one process: each of `world` ranks
    decodes its token chunks (rdkv_cuda_decode_partial), the stacked partials
    are merged (rdkv_cuda_decode_merge) — equal to the one-rank decode."""
    rng = np.random.default_rng(200 + world + appends)
    cases = []
    for n in (20, 128, 161, 400, 900):
        k, v, vb, kb, q = _random_case(rng, 1000, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(1000, n, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, 4, io=io, appends=appends, rng=rng, tol=U2X_TOL)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).to(io)
    want = P.packed_decode_step(model, q).float()
    parts = torch.stack([P.decode_partial(model, q, r, world) for r in range(world)])
    got = P.merge_partials(parts, io).float()
    ref = P.merge_partials_reference(parts).float()
    assert float(((got - ref).norm(dim=-1) / ref.norm(dim=-1)).max()) < (1e-5 if io == torch.float32 else 1e-3)
    err = (got - want).norm(dim=-1) / want.norm(dim=-1)
    assert float(err.max()) < (2 * U2X_TOL if io == torch.float32 else 2e-3), float(err.max())



@pytest.mark.parametrize("g,io", [(4, torch.float32), (4, torch.float16), (8, torch.float32), (2, torch.float16),
                                  (8, torch.float16), (6, torch.float32)])
def test_mix_mostly_two_bit_tiles(cuda, orc, g, io):
    """Heavy-hitter shape on the fast kernel (MIX): tiles with up to 8 4-bit V
    rows and up to 28 4-bit K channels next to uniform 2-bit tiles."""
    rng = np.random.default_rng(300 + g)
    cases = []
    for i, n in enumerate((5, 40, 97, 128, 133, 150, 60, 128)):
        k, v, vb, kb, q = _random_case(rng, 400, g)
        vb[:] = 0
        kept = np.sort(rng.choice(400, n, replace=False))
        vb[kept] = 2
        kb[:] = 2
        if i % 2 == 1:
            r4 = min(n - 1, int(rng.integers(1, 17)))
            vb[kept[rng.choice(n, r4, replace=False)]] = 4
        if i % 3 != 2:
            kb[rng.choice(D, int(rng.integers(1, 29)), replace=False)] = 4
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, g, io=io, tol=U2X_TOL)
    assert model.plan.uniform2 == 3, model.plan.uniform2
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst


@pytest.mark.parametrize("g,T,io,nkept", [(4, 700, torch.float32, 300), (7, 2000, torch.float16, 1500),
                                          (4, 3000, torch.float16, 2600), (8, 400, torch.float32, 90)])
def test_mixed_248_split_k_kernel(cuda, orc, g, T, io, nkept):
    """Every class the chunked split-K kernel (decode_u24) handles — V rows and K channels
    at 2, 4 and 8 bits (no Zone B / k16), short and long tiles, GQA 4 / 7 / 8 — against
    the oracle, with and without the split-K partials workspace."""
    rng = np.random.default_rng(300 + g + T)
    cases = []
    for i in range(6):
        k, v, vb, kb, q = _random_case(rng, T, g)
        vb[:] = 0
        kept = np.sort(rng.choice(T, max(8, nkept - (nkept // 8) * i), replace=False))
        vb[kept] = rng.choice([2, 4, 8], kept.size, p=[0.6, 0.3, 0.1])
        kb[:] = rng.choice([0, 2, 4, 8], D, p=[0.05, 0.55, 0.3, 0.1])
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, g, io=io, rng=rng, tol=U2X_TOL)
    assert model.plan.mix24 and not model.plan.uniform2
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst
    qd = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).to(io)
    split = P.packed_decode_step(model, qd).float()
    ws, model.split_ws = model.split_ws, None
    whole = P.packed_decode_step(model, qd).float()
    model.split_ws = ws
    assert float(((split - whole).norm() / whole.norm()).item()) < 1e-3


@pytest.mark.parametrize("g,appends,io", [(4, 1, torch.float16), (4, 7, torch.float32), (8, 3, torch.float16),
                                          (7, 20, torch.float32), (4, 33, torch.float16)])
def test_zone_c_prepass_matches_fused_and_oracle(cuda, orc, g, appends, io):
    """Zone C through the prepass (zc_partial_kernel: one warp per unit folds the appended
    rows into a [g][d + 2] softmax row, the short-tile kernel merges it in its epilogue) —
    the default whenever the model carries its Zone C workspace — against the oracle, the
    fused / chunked variants (no workspace) and the bound-less path."""
    rng = np.random.default_rng(700 + 10 * g + appends)
    cases = []
    for n in (1, 40, 128, 150, 160, 96):
        k, v, vb, kb, q = _random_case(rng, 500, g)
        vb[:] = 0
        vb[np.sort(rng.choice(500, n, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    worst, model = _run_batch(cuda, orc, cases, g, io=io, appends=appends, rng=rng, tol=U2X_TOL)
    assert model.plan.uniform2 == 2 and model.zc_ws is not None
    assert worst < (U2X_TOL if io == torch.float32 else 1e-3), worst
    q = torch.from_numpy(np.stack([c[4] for c in cases])).to(cuda).to(io)
    tiny = torch.empty(1, dtype=torch.uint8, device=cuda)  # too small: no prepass
    count, model.zc_count = model.zc_count, None
    pre = P.packed_decode_step(model, q).float()  # no host bound: the prepass
    chunked = P.packed_decode_step(model, q, workspace=tiny).float()  # chunked Zone C
    model.zc_count = count
    dflt = P.packed_decode_step(model, q).float()  # bound known: fused (<= 4 rows) or prepass
    fused = P.packed_decode_step(model, q, workspace=tiny).float()
    for other in (fused, chunked, dflt):
        assert float(((pre - other).norm() / other.norm()).item()) < 1e-3
    if appends > 4:
        assert torch.equal(pre, dflt)  # the same prepass path, bound or not
