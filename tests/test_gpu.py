"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on the same seeded
inputs and weights.

Tolerances (BASELINE.json north_star):
  FP32 mode: logits / incoming messages within 1e-3 relative (to max |value|); decoded grids,
             first-reveal counts, remask rows / steps / indices identical.
  BF16 mode: logits / messages within 1e-2 relative (bf16 operands, fp32 accumulation, tanh-form
             GELU in the fused MLP epilogues). Decisions at the BASELINE shapes are checked
             teacher-forced in test_gpu_parity.py.
"""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-3
BF16_TOL = 1e-2


def ctx_for(P, model, wl, seed=1, edges=None):
    e = wl.code() if edges is None else edges
    w = P.weights_init(model, seed)
    return P.Context(model, w, e, wl.checks, wl.slots), e, w


def as_run(P, model, w):
    return P.model_weights_as_run(model, w)


# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_denoise_parity_all_configs(P, oracle, parity_report, name):
    """One forward on partially revealed grids: logits and every layer's check messages."""
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    ctx, e, w = ctx_for(P, model, wl)
    nb = 2 if name in ("c1", "c2") else 1
    _, S = wl.bins(e, 0, nb)
    rng = np.random.default_rng(11)
    X = np.where(rng.random((nb, wl.k, wl.slots)) < 0.5, rng.integers(0, model.q, size=(nb, wl.k, wl.slots)), -1)
    X = X.astype(np.int32)
    lg, inc = ctx.denoise(X, S, want_incoming=True)
    tol = FP32_TOL if model.precision == P.FP32 else BF16_TOL
    errs = []
    for b in range(nb):
        lo, io = oracle.denoise(model, as_run(P, model, w), e, wl.checks, wl.slots, X[b], S[b].astype(np.float64), True)
        errs.append(rel_err(lg[b], lo))
        errs.extend(rel_err(inc[b, layer], io[layer]) for layer in range(model.layers))
    parity_report[f"denoise_{name}"] = {"max_rel_err": max(errs), "tol": tol}
    assert max(errs) < tol, errs


def test_c1_full_decode_identical_to_oracle(P, oracle):
    """BASELINE config 1 end to end (64 bins, T=4, FP32): identical decoded sets and SER."""
    cfg = P.configs()["c1"]
    wl, model = cfg.workload, cfg.model
    ctx, e, w = ctx_for(P, model, wl)
    truth, S = wl.bins(e, 0, cfg.bins)
    sched = P.RevealSchedule(steps=cfg.steps)
    grid, fl, tr = ctx.refine(S, wl.k, sched, want_final_logits=True, want_trace=True)
    ro = oracle.refine(model, as_run(P, model, w), e, wl.checks, wl.slots, S.astype(np.float64), wl.k, sched,
                       want_final_logits=True)
    assert np.array_equal(grid, ro["grid"])
    assert rel_err(fl, ro["final_logits"]) < FP32_TOL
    assert np.array_equal(tr["first_reveals"], ro["first_reveals"])
    assert P.ser_cer(truth, grid) == P.ser_cer(truth, ro["grid"])


@pytest.mark.parametrize("remask", ["thr", "rank"])
def test_remask_indices_identical_fp32(P, oracle, remask):
    """Quality-guided remasking (refine.cpp:238-292): same rows selected, same T_rm, same grids;
    rows outside K_low stay bit-identical."""
    wl = P.Workload(m=4, slots=16, checks=8, k=8, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=4, dim=32, hidden=64, layers=2, heads=2)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 6)
    rm = P.RemaskConfig(thresholds=(0.3, 0.2, 0.1)) if remask == "thr" else P.RemaskConfig(rank_fraction=0.25)
    sched = P.RevealSchedule(steps=6)
    grid, fl, tr = ctx.refine(S, 8, sched, rm, want_final_logits=True, want_trace=True)
    ro = oracle.refine(model, as_run(P, model, w), e, wl.checks, wl.slots, S.astype(np.float64), 8, sched, rm,
                       want_final_logits=True)
    assert np.array_equal(grid, ro["grid"])
    assert np.array_equal(tr["remask_rows"], ro["remask_rows"])
    assert np.array_equal(tr["remask_steps"], ro["remask_steps"])
    assert np.array_equal(tr["remask_mask"], ro["remask_mask"])
    assert rel_err(fl, ro["final_logits"]) < FP32_TOL
    plain = ctx.refine(S, 8, sched)
    keep = tr["remask_mask"] == 0
    assert np.array_equal(grid[keep], plain[keep])


def test_threshold_remask_buckets_with_mixed_row_counts(P, oracle):
    """Thresholds that select different |K_low| per bin exercise the per-bucket sub-batches."""
    wl = P.Workload(m=4, slots=16, checks=8, k=4, snr_db=4.0)
    model = P.Model.ref_exact(4, 32)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 8)
    sched = P.RevealSchedule(steps=5)
    ro0 = oracle.refine(model, as_run(P, model, w), e, wl.checks, wl.slots, S.astype(np.float64), 4, sched,
                        want_final_logits=True)
    conf = np.stack([(1.0 / np.exp(f - f.max(-1, keepdims=True)).sum(-1)).mean(-1) for f in ro0["final_logits"]])
    thr = float(np.median(conf))
    rm = P.RemaskConfig(thresholds=(min(0.99, thr + 1e-4), thr * 0.99))
    grid, tr = ctx.refine(S, 4, sched, rm, want_trace=True)
    ro = oracle.refine(model, as_run(P, model, w), e, wl.checks, wl.slots, S.astype(np.float64), 4, sched, rm)
    assert len(set(ro["remask_rows"][:, 0].tolist())) > 1
    assert np.array_equal(grid, ro["grid"])
    assert np.array_equal(tr["remask_rows"], ro["remask_rows"])
    assert np.array_equal(tr["remask_mask"], ro["remask_mask"])


# ---- invariants on the device ------------------------------------------------------------------
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_device_row_permutation_equivariance_bitwise(P, prec):
    wl = P.Workload(m=6, slots=16, checks=8, k=4, snr_db=6.0)
    model = P.Model(m=6, dim=64, hidden=128, layers=2, heads=2, precision=P.FP32 if prec == "fp32" else P.BF16)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 1)
    X = np.random.default_rng(1).integers(-1, 64, size=(1, 4, 16)).astype(np.int32)
    X[0, 3] = X[0, 1]  # two identical rows -> exact ties
    base = ctx.denoise(X, S)
    p = [2, 0, 3, 1]
    perm = ctx.denoise(X[:, p], S)
    assert np.array_equal(perm, base[:, p])
    assert np.array_equal(base[0, 1], base[0, 3])


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_device_extrinsicity_bitwise(P, prec):
    wl = P.Workload(m=6, slots=16, checks=8, k=2, snr_db=6.0)
    model = P.Model(m=6, dim=64, hidden=64, layers=1, precision=P.FP32 if prec == "fp32" else P.BF16)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 1)
    X = np.random.default_rng(2).integers(-1, 64, size=(1, 2, 16)).astype(np.int32)
    _, base = ctx.denoise(X, S, want_incoming=True)
    for l in (0, 7, 15):
        Y = X.copy()
        Y[0, :, l] = (np.maximum(Y[0, :, l], 0) + 5) % 64
        _, inc = ctx.denoise(Y, S, want_incoming=True)
        assert np.array_equal(inc[0, 0][:, l], base[0, 0][:, l])


def test_determinism_and_chunk_invariance(P):
    """Run-to-run bitwise determinism (no atomics) and independence of the internal chunking."""
    cfg = P.configs()["c2"]
    wl = cfg.workload
    model = P.Model(m=6, dim=64, hidden=128, layers=2, heads=2, precision=P.BF16)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 37)
    sched = P.RevealSchedule(steps=5)
    a = ctx.refine(S, wl.k, sched, P.RemaskConfig(rank_fraction=0.25))
    b = ctx.refine(S, wl.k, sched, P.RemaskConfig(rank_fraction=0.25))
    ctx.set_chunk(5)
    c = ctx.refine(S, wl.k, sched, P.RemaskConfig(rank_fraction=0.25))
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_c2_full_size_properties(P):
    """BASELINE config 2 at full size (4096 bins, bf16): valid symbols, determinism, and the
    decode is invariant to the bin batching (a checksum of per-bin checksums)."""
    cfg = P.configs()["c2"]
    wl, model = cfg.workload, cfg.model
    ctx, e, w = ctx_for(P, model, wl)
    truth, S = wl.bins(e, 0, cfg.bins)
    sched = P.RevealSchedule(steps=cfg.steps)
    g = ctx.refine(S, wl.k, sched)
    assert np.all((g >= 0) & (g < model.q))
    half = ctx.refine(S[: cfg.bins // 2], wl.k, sched)
    assert np.array_equal(half, g[: cfg.bins // 2])
    sums = (g.astype(np.int64) * np.arange(1, wl.k * wl.slots + 1).reshape(wl.k, wl.slots)).sum((1, 2))
    g2 = ctx.refine(S, wl.k, sched)
    sums2 = (g2.astype(np.int64) * np.arange(1, wl.k * wl.slots + 1).reshape(wl.k, wl.slots)).sum((1, 2))
    assert int(sums.sum()) == int(sums2.sum())
    ser, cer = P.ser_cer(truth, g)
    assert 0.0 <= ser <= 1.0 and 0.0 <= cer <= 1.0


def test_c3_full_size_properties(P):
    """BASELINE config 3 at full size (16384 bins, N=6, D=256, H=1024, 8 heads, T=16 + rank-25%
    remasking, bf16 — the bench's kernel set over several device chunks): valid symbols, and a
    re-decode of the first 3000 bins in 700-bin chunks (different chunk boundaries, eager and graph
    runs) reproduces them exactly."""
    cfg = P.configs()["c3"]
    wl, model = cfg.workload, cfg.model
    ctx, e, w = ctx_for(P, model, wl)
    truth, S = wl.bins(e, 0, cfg.bins)
    sched = P.RevealSchedule(steps=cfg.steps)
    g = ctx.refine(S, wl.k, sched, cfg.remask)
    assert g.shape == (cfg.bins, wl.k, wl.slots) and np.all((g >= 0) & (g < model.q))
    ctx.set_chunk(700)
    part = ctx.refine(S[:3000], wl.k, sched, cfg.remask)
    assert np.array_equal(part, g[:3000])
    ser, cer = P.ser_cer(truth[:64], g[:64])
    assert 0.0 <= ser <= 1.0 and 0.0 <= cer <= 1.0


# ---- edge cases ---------------------------------------------------------------------------------
def test_edge_shapes_and_schedules(P, oracle):
    wl = P.Workload(m=4, slots=16, checks=8, k=3, snr_db=6.0)
    model = P.Model.ref_exact(4, 32)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 3)
    wr = as_run(P, model, w)
    for K, sched in [(1, P.RevealSchedule(steps=3)), (3, P.RevealSchedule(steps=1)),
                     (3, P.RevealSchedule(steps=4, first_reveal=False)),
                     (3, P.RevealSchedule(steps=6, tau_max=2.0, tau_min=0.25))]:
        g = ctx.refine(S, K, sched)
        ro = oracle.refine(model, wr, e, wl.checks, wl.slots, S.astype(np.float64), K, sched)
        assert np.array_equal(g, ro["grid"]), (K, sched)
    assert ctx.refine(S[:0], 3, P.RevealSchedule(steps=2)).shape == (0, 3, 16)


def test_sparse_graph_slots_without_checks(P, oracle):
    """test_denoiser.cpp:249-267: slots with no incident check get zero messages."""
    model = P.Model.ref_exact(4, 32)
    edges = np.array([[0, 0, 3], [0, 1, 5]], np.int32)
    w = P.weights_init(model, 1)
    ctx = P.Context(model, w, edges, 1, 12)
    S = np.log(np.full((1, 12, 16), 1.0 / 16, np.float32))
    X = np.random.default_rng(0).integers(-1, 16, size=(1, 2, 12)).astype(np.int32)
    lg, inc = ctx.denoise(X, S, want_incoming=True)
    lo, io = oracle.denoise(model, as_run(P, model, w), edges, 1, 12, X[0], S[0].astype(np.float64), True)
    assert rel_err(lg[0], lo) < FP32_TOL
    assert np.all(inc[0, 0][:, 2:] == 0.0)


def test_input_errors_surface_like_the_reference(P):
    wl = P.Workload(m=4, slots=16, checks=8, k=2, snr_db=6.0)
    model = P.Model.ref_exact(4, 32)
    ctx, e, w = ctx_for(P, model, wl)
    _, S = wl.bins(e, 0, 1)
    with pytest.raises(ValueError, match="embed_grid: token out of range"):
        ctx.denoise(np.full((1, 2, 16), 16, np.int32), S)
    with pytest.raises(ValueError, match="strictly descending"):
        ctx.refine(S, 2, P.RevealSchedule(steps=2), P.RemaskConfig(thresholds=(0.4, 0.6)))
    with pytest.raises(ValueError, match="tau_max >= tau_min > 0"):
        ctx.refine(S, 2, P.RevealSchedule(steps=2, tau_max=0.5, tau_min=1.0))
    with pytest.raises(ValueError, match="need T >= 1"):
        ctx.refine(S, 2, P.RevealSchedule(steps=0))


def test_reference_engine_with_gpu_denoiser():
    """The drop-in boundary end to end: the reference's own ura::run_refinement /
    run_with_remasking driving cider::GpuStructuredDenoiser (include/cider_ura.hpp), the device
    loop, and a BinDecoder — identical grids to the reference (oracle/adapter_test.cpp)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "adapter_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/adapter_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("m,d", [(4, 3), (6, 5), (6, 6), (8, 6)])
def test_wht_check_update_matches_reference_vectors(P, oracle, m, d):
    """batched WHT-domain GF(Q) check update on the device vs the oracle's
    restatement of check_update_wht (bp.cpp:128-149; pinned to the reference by test_oracle.py),
    within the reference's own WHT-vs-direct tolerance (test_bp.cpp:145-168: 1e-8)."""
    q = 1 << m
    rng = np.random.default_rng(m * 10 + d)
    n = 64
    v2c = rng.random((n, d, q)) ** 3
    v2c /= v2c.sum(-1, keepdims=True)
    cf = rng.integers(1, q, size=(n, d)).astype(np.int32)
    out = P.check_update_wht(m, v2c, cf)
    for c in range(0, n, 7):
        for i in range(d):
            others = [j for j in range(d) if j != i]
            ref = oracle.check_update_wht(m, v2c[c, others], cf[c, others], int(cf[c, i]))
            assert np.abs(out[c, i] - ref).max() < 1e-8
    assert np.allclose(out.sum(-1), 1.0)


# ---- batched GF(Q) FFT-BP decoder -----------------------------------------------
def _slot_beliefs(S):
    """bp.cpp:61-77 (per-slot softmax of the evidence rows)."""
    x = np.exp(S - S.max(-1, keepdims=True))
    return x / x.sum(-1, keepdims=True)


@pytest.mark.parametrize("name,nb", [("c1", 16), ("c2", 8), ("c3", 2)])
def test_bp_decode_matches_reference(P, reference, name, nb):
    """Device bp_decode vs the reference's (bp.cpp:271-347, WHT backend; long double spectra) on
    the config's code and seeded evidence: identical hard decisions, convergence flags and
    iteration counts; marginals within 1e-9 (the device keeps the spectra in double-double)."""
    wl = P.configs()[name].workload
    e = wl.code()
    _, S = wl.bins(e, 0, nb)
    lam = _slot_beliefs(S.astype(np.float64))
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    cfg = P.BpConfig(max_iters=30)
    hard, marg, conv, its = dec.bp_decode(lam, cfg)
    rh, rm, rc, ri = reference.bp_decode(wl.m, e, wl.checks, wl.slots, lam, max_iters=30)
    assert np.array_equal(hard, rh)
    assert np.array_equal(conv, rc.astype(bool))
    assert np.array_equal(its, ri)
    assert rel_err(marg, rm) < 1e-9


@pytest.mark.parametrize("name,nb", [("c1", 16), ("c2", 6)])
def test_sic_decode_matches_reference(P, reference, name, nb):
    """Device sic_decode (bp.cpp:349-368): K BP stages with cancellation at log(K/Q); the decoded
    grid (rows in decode order) and per-stage convergence / iteration counts match the reference."""
    wl = P.configs()[name].workload
    e = wl.code()
    _, S = wl.bins(e, 0, nb)
    S = S.astype(np.float64)
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    cfg = P.BpConfig(max_iters=20)
    grid, sc, si = dec.sic_decode(S, wl.k, cfg)
    rg, rsc, rsi = reference.sic_decode(wl.m, e, wl.checks, wl.slots, S, wl.k, max_iters=20)
    assert np.array_equal(grid, rg)
    assert np.array_equal(sc, rsc.astype(bool))
    assert np.array_equal(si, rsi)


def test_bp_early_exit_freezes_converged_bins(P, reference):
    """A bin whose evidence is one clean codeword converges at iteration 1 and stays frozen while
    noisy bins of the same batch keep iterating (per-bin control flow of bp.cpp:315-318)."""
    wl = P.configs()["c2"].workload
    e = wl.code()
    truth, S = wl.bins(e, 0, 4)
    q = 1 << wl.m
    clean = np.full((wl.slots, q), -30.0)
    clean[np.arange(wl.slots), truth[0, 0]] = 0.0
    S = S.astype(np.float64)
    S[0] = clean
    lam = _slot_beliefs(S)
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    hard, marg, conv, its = dec.bp_decode(lam, P.BpConfig(max_iters=25))
    rh, rm, rc, ri = reference.bp_decode(wl.m, e, wl.checks, wl.slots, lam, max_iters=25)
    assert conv[0] and its[0] == 1 and np.array_equal(hard[0], truth[0, 0])
    assert np.array_equal(hard, rh) and np.array_equal(its, ri)


def test_bp_errors_like_the_reference(P):
    wl = P.configs()["c1"].workload
    e = wl.code()
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    lam = np.full((1, wl.slots, 16), 1.0 / 16)
    with pytest.raises(ValueError, match="max_iters"):
        dec.bp_decode(lam, P.BpConfig(max_iters=0))
    with pytest.raises(ValueError, match="message_floor"):
        dec.bp_decode(lam, P.BpConfig(message_floor=0.0))
    with pytest.raises(ValueError, match="K >= 1"):
        dec.sic_decode(np.zeros((1, wl.slots, 16)), 0)


# ---- the BASELINE evidence generator on the device --------------------------------
@pytest.mark.parametrize("name,first,n", [("c1", 0, 64), ("c2", 7, 48), ("c3", 3, 12), ("c4", 0, 6), ("c5", 100, 8)])
def test_device_workload_matches_host_generator(P, name, first, n):
    """Device bins (one thread per bin, mt19937_64 + the libstdc++ distributions restated) vs the
    host generator: identical codewords; S identical except where a double exp/log differs from
    glibc in the last ulp (then within one float ulp)."""
    cfg = P.configs()[name]
    wl = cfg.workload
    e = wl.code()
    ctx = P.Context(P.Model(m=wl.m, dim=64, hidden=64, precision=P.FP32), P.weights_init(P.Model(m=wl.m, dim=64, hidden=64), 1),
                    e, wl.checks, wl.slots)
    th, Sh = wl.bins(e, first, n)
    td, Sd = wl.bins_device(ctx, e, first, n)
    assert np.array_equal(th, td)
    diff = Sd != Sh
    assert diff.mean() < 1e-4
    assert np.all(np.abs(Sd - Sh) <= np.spacing(np.abs(Sh)) * 1.0001)


# ---- ragged per-bin loads (protocol bins carry K_chi in 1..k_max) -----------------
def test_refine_ragged_equals_per_load_calls(P):
    """cider_refine_ragged buckets bins by load and runs each bucket with its own schedule / remask
    (a DecoderBank's per-load configs); every bin's grid equals a uniform-K call on that bin."""
    cfg = P.configs()["c2"]
    wl = cfg.workload
    e = wl.code()
    model = P.Model(m=wl.m, dim=64, hidden=128, layers=1, heads=2, precision=P.FP32)
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    rng = np.random.default_rng(5)
    loads = rng.integers(1, 5, size=12).astype(np.int32)
    _, S = wl.bins(e, 0, 12)
    scheds = [P.RevealSchedule(steps=2 + k) for k in range(4)]
    rms = [None, P.RemaskConfig(thresholds=[0.5]), None, P.RemaskConfig(thresholds=[0.6, 0.3])]
    grids = ctx.refine_ragged(S, loads, scheds, rms)
    for b in range(12):
        k = int(loads[b])
        ref = ctx.refine(S[b:b + 1], k, scheds[k - 1], rms[k - 1])
        assert grids[b].shape == (k, wl.slots) and np.array_equal(grids[b], ref[0])
    with pytest.raises(ValueError, match="load outside"):
        ctx.refine_ragged(S[:1], np.array([5], np.int32), scheds, rms)


# ---- the fused sm_100a kernels of the BASELINE c3/c5 shapes (Q = D = 256, heads = 8, degree 6) ---
@pytest.mark.parametrize("k,dim", [(4, 256), (8, 256), (4, 128)])
def test_fused_bf16_kernels_parity_and_invariants(P, oracle, k, dim):
    """The c3/c5 kernel set — Lambda-bar -> demix -> e in one 2-SM kernel, the 2-SM MLPs with
    X-staged TMA-stored outputs, the one-pass attention pool, the lap-scheduled normalise and the
    CTA-pair message GEMMs — on a small code: parity with the oracle, bitwise row-permutation
    equivariance and bitwise extrinsicity of the layer's check messages (SURVEY §4 property tests,
    test_denoiser.cpp:213-247, 293-326). 40 bins: an odd number of 128-row tiles for K = 8 (the
    CTA pair's second m-tile falls past the bins)."""
    wl = P.Workload(m=8, slots=16, checks=8, k=k, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=8, dim=dim, hidden=256, layers=1, heads=8, precision=P.BF16)
    ctx, e, w = ctx_for(P, model, wl)
    nb = 40
    _, S = wl.bins(e, 0, nb)
    rng = np.random.default_rng(5)
    X = np.where(rng.random((nb, k, wl.slots)) < 0.5, rng.integers(0, model.q, size=(nb, k, wl.slots)), -1).astype(np.int32)
    X[:, k - 1] = X[:, 0]  # identical rows -> exact ties
    ctx.reset_stats()
    ctx.set_profiling(True)
    lg, inc = ctx.denoise(X, S, want_incoming=True)
    ctx.set_profiling(False)
    tags = set(ctx.kernel_stats())
    want = {"mlp_gate", "pool_attn", "mlp_agg", "mlp_fuse"}
    if dim == 256:
        want |= {"demix_evid", "grp_normalise", "grp_message"}
    assert want <= tags, tags
    wr = as_run(P, model, w)
    for b in (0, nb - 1):
        lo, io = oracle.denoise(model, wr, e, wl.checks, wl.slots, X[b], S[b].astype(np.float64), True)
        assert rel_err(lg[b], lo) < BF16_TOL
        assert rel_err(inc[b, 0], io[0]) < BF16_TOL
    assert np.array_equal(lg[:, k - 1], lg[:, 0])
    p = np.roll(np.arange(k), 1)
    lgp = ctx.denoise(X[:, p], S)
    assert np.array_equal(lgp, lg[:, p])
    # every slot in turn, and a second token change: the leave-one-out softmax must be the same function of the
    # other edges whether or not the changed slot's own score is the check's largest (pool_mma.cuh, row i1)
    for l in range(wl.slots):
        for add in (7, 101):
            Y = X.copy()
            Y[:, :, l] = (np.maximum(Y[:, :, l], 0) + add) % model.q
            _, inc2 = ctx.denoise(Y, S, want_incoming=True)
            assert np.array_equal(inc2[:, 0][:, :, l], inc[:, 0][:, :, l]), (l, add)
