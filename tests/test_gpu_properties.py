"""The reference's own hot-path property tests (SURVEY §4 ★: test_denoiser.cpp, test_refine.cpp) run on
the device kernels, in FP32 parity mode and through the BF16 tcgen05 kernel set at the BASELINE c3 / c5
shapes. They need no oracle: each is an exact (bitwise or closed-form) property of the math.

* gates forced open / closed give exact pass-through (test_denoiser.cpp:141-159) and, with Module B's
  fusion zeroed, the denoiser is site-local (test_denoiser.cpp:46-68);
* the demix responsibilities sum to one over the rows: sum_k e[k, l] = S[l] V (test_denoiser.cpp:70-139);
* first reveal = one site per slot, the reveal target is honoured, all sites are revealed by step T
  (test_refine.cpp:110-146, 176-202);
* T = 1 makes two denoiser calls, the last one the gamma = 0 pass (test_refine.cpp:164-174);
* remasking clamps the rows it does not re-decode bit for bit (test_refine.cpp:262-298).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def layer_offsets(model):
    """Offsets into the flat weight vector (cider.h: embed | out_proj | sym_embed | per layer gate_a,
    check_agg, fuse_b as {w1, b1, w2, b2} | per-layer attention)."""
    Q, D, H = model.q, model.dim, model.hidden
    off = {"embed": 0, "out_proj": (Q + 1) * D, "sym_embed": (Q + 1) * D + Q * D}
    o = (Q + 1) * D + 2 * Q * D
    layers = []
    for _ in range(model.layers):
        lay = {}
        for name, kin in (("gate_a", 2 * D), ("check_agg", D), ("fuse_b", 2 * D)):
            lay[name] = {"w1": o, "b1": o + H * kin, "w2": o + H * kin + H, "b2": o + H * kin + H + D * H}
            o += H * kin + H + D * H + D
        layers.append(lay)
    off["layers"] = layers
    off["end_maps"] = o
    return off


def forced_gate_weights(P, model, gate_bias):
    """Every layer: gate_a's output layer = (0, gate_bias) so that g = sigmoid(gate_bias) everywhere, and
    fuse_b's output layer = 0 so that Module B adds nothing (Z-hat = z~)."""
    w = P.weights_init(model, 1)
    off = layer_offsets(model)
    assert off["end_maps"] <= w.size
    D, H = model.dim, model.hidden
    for lay in off["layers"]:
        g, f = lay["gate_a"], lay["fuse_b"]
        w[g["w2"]: g["w2"] + D * H] = 0.0
        w[g["b2"]: g["b2"] + D] = gate_bias
        w[f["w2"]: f["w2"] + D * H] = 0.0
        w[f["b2"]: f["b2"] + D] = 0.0
    return w, off


MODELS = {
    "fp32": dict(m=4, dim=32, hidden=64, layers=2, heads=2, k=3, slots=16, checks=8, bins=3),
    # the bench's kernel set: Q = D = 256, 8 heads, K = 8, degree-6 checks; 40 bins = 2 gate tiles per pair-round
    "bf16_c3": dict(m=8, dim=256, hidden=1024, layers=2, heads=8, k=8, slots=64, checks=32, bins=40),
    "bf16_c2": dict(m=6, dim=128, hidden=512, layers=2, heads=8, k=4, slots=32, checks=16, bins=24),
}


def setup(P, name, gate_bias):
    s = MODELS[name]
    prec = P.FP32 if name == "fp32" else P.BF16
    model = P.Model(m=s["m"], dim=s["dim"], hidden=s["hidden"], layers=s["layers"], heads=s["heads"], precision=prec)
    wl = P.Workload(m=s["m"], slots=s["slots"], checks=s["checks"], k=s["k"], snr_db=4.0, p_erase=0.1, p_false=0.1)
    e = wl.code()
    w, off = forced_gate_weights(P, model, gate_bias)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, s["bins"])
    rng = np.random.default_rng(11)
    X = rng.integers(0, model.q, size=(s["bins"], s["k"], s["slots"]))
    X = np.where(rng.random(X.shape) < 0.4, -1, X).astype(np.int32)
    return model, wl, ctx, w, off, S, X


@pytest.mark.parametrize("name", ["fp32", "bf16_c3", "bf16_c2"])
def test_gate_forced_open_is_exact_pass_through_and_site_local(P, name):
    """g = 1: z~ = Z whatever the evidence says (test_denoiser.cpp:141-159), so with the fusion zeroed the
    logits are E[X] W^T: independent of S bit for bit, equal to the closed form, and site-local
    (test_denoiser.cpp:46-68: a changed token changes its own site only)."""
    model, wl, ctx, w, off, S, X = setup(P, name, +1000.0)
    lg = ctx.denoise(X, S)
    S2 = np.roll(S, 1, axis=0) * 0.5 + 0.25
    assert np.array_equal(lg, ctx.denoise(X, S2))
    wr = P.model_weights_as_run(model, w)
    Q, D = model.q, model.dim
    E = wr[: (Q + 1) * D].reshape(Q + 1, D)
    W = wr[off["out_proj"]: off["out_proj"] + Q * D].reshape(Q, D)
    want = E[np.where(X < 0, Q, X)] @ W.T
    err = np.abs(lg - want).max() / np.abs(want).max()
    assert err < 1e-5, err  # operands are exact in both modes; only the fp32 accumulation differs
    Y = X.copy()
    b, k, l = 1, 1, 5
    Y[b, k, l] = (max(int(Y[b, k, l]), 0) + 3) % Q
    lg2 = ctx.denoise(Y, S)
    same = np.ones(X.shape, bool)
    same[b, k, l] = False
    assert np.array_equal(lg2[same], lg[same])
    assert not np.array_equal(lg2[b, k, l], lg[b, k, l])


@pytest.mark.parametrize("name", ["fp32", "bf16_c3", "bf16_c2"])
def test_gate_forced_closed_passes_the_evidence_embedding(P, name):
    """g = 0: z~ = e (test_denoiser.cpp:141-159). e = sum_a r_a S_la v_a vanishes where the slot's evidence
    row is zero, so those sites' logits are exactly 0 for every row and every token; and a slot's e row
    does not depend on the tokens of other slots."""
    model, wl, ctx, w, off, S, X = setup(P, name, -1000.0)
    S = S.copy()
    dead = [2, 7]
    S[:, dead, :] = 0.0
    lg = ctx.denoise(X, S)
    assert np.all(lg[:, :, dead, :] == 0.0)
    live = [l for l in range(wl.slots) if l not in dead]
    assert np.abs(lg[:, :, live, :]).max() > 0.0
    Y = X.copy()
    Y[:, :, 9] = (np.maximum(Y[:, :, 9], 0) + 1) % model.q
    lg2 = ctx.denoise(Y, S)
    keep = [l for l in range(wl.slots) if l != 9]
    assert np.array_equal(lg2[:, :, keep, :], lg[:, :, keep, :])


@pytest.mark.parametrize("name", ["fp32", "bf16_c3", "bf16_c2"])
def test_responsibilities_sum_to_one_over_the_rows(P, name):
    """test_denoiser.cpp:70-104 (normalisation) + 106-139 (evidence embedding) through the fused kernels: with
    the gate closed the logits are e W^T, and since sum_k r[k, l, a] = 1 the row sum of e is S[l] V whatever
    the tokens are: sum_k logits[k, l, :] = (S[l] V) W^T."""
    model, wl, ctx, w, off, S, X = setup(P, name, -1000.0)
    lg = ctx.denoise(X, S).astype(np.float64)
    wr = P.model_weights_as_run(model, w)
    Q, D = model.q, model.dim
    W = wr[off["out_proj"]: off["out_proj"] + Q * D].reshape(Q, D)
    V = wr[off["sym_embed"]: off["sym_embed"] + Q * D].reshape(Q, D)
    want = (S.astype(np.float64) @ V) @ W.T  # B x L x Q
    got = lg.sum(axis=1)
    err = np.abs(got - want).max() / np.abs(want).max()
    print(name, "row-sum rel err", err)
    assert err < (1e-4 if name == "fp32" else 1e-2), err


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_reveal_schedule_properties_at_baseline_shapes(P, name):
    """test_refine.cpp:110-146, 176-202 on the device loop at the BASELINE shapes (bf16, 96 bins): the first
    step reveals exactly one site per slot, the per-step counts never exceed what is masked, and step T
    reveals everything that is left (rho(T) = 1)."""
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    nb = 96
    _, S = wl.bins(e, 0, nb)
    sched = P.RevealSchedule(steps=cfg.steps)
    grid, tr = ctx.refine(S, wl.k, sched, want_trace=True)
    n = wl.k * wl.slots
    assert np.all(tr["n_passes"] == 1) and np.all(tr["n_reveal_counts"] == cfg.steps)
    assert np.all(tr["first_reveals"] == wl.slots)
    sites = tr["first_step_sites"].astype(np.int64)
    assert np.all(sites.sum(axis=1) == 1)  # one row per slot (B x K x L summed over the rows)
    counts = tr["reveal_counts"][:, : cfg.steps].astype(np.int64)
    assert np.all(counts >= 0) and np.all(counts[:, 0] == wl.slots)
    cum = counts.cumsum(axis=1)
    assert np.all(cum[:, -1] == n)
    # cumulative cosine target: after step t at least round-down of rho(t) n sites are revealed
    rho = 0.5 * (1.0 - np.cos(np.pi * np.arange(1, cfg.steps + 1) / cfg.steps))
    assert np.all(cum >= np.floor(rho * n - 1e-9)[None, :] - 1)
    assert np.all(cum[:, 1:] <= np.maximum(np.ceil(rho * n)[None, 1:] + 1, wl.slots))
    assert np.all((grid >= 0) & (grid < model.q))


def test_single_step_schedule_makes_two_denoiser_calls(P):
    """test_refine.cpp:164-174: T = 1 = one masked-loop forward + the gamma = 0 pass."""
    wl = P.Workload(m=6, slots=32, checks=16, k=4, snr_db=6.0)
    model = P.Model(m=6, dim=128, hidden=512, layers=2, heads=8, precision=P.BF16)
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 8)
    ctx.set_profiling(True)
    for steps, forwards in ((1, 2), (3, 4)):
        ctx.reset_stats()
        ctx.refine(S, wl.k, P.RevealSchedule(steps=steps))
        st = ctx.kernel_stats()
        assert st["gemm_logits"]["launches"] == forwards, st["gemm_logits"]
        assert st["mlp_agg"]["launches"] == forwards * model.layers


@pytest.mark.parametrize("name,nb", [("c3", 300), ("c2", 1000)])
def test_remasking_clamps_the_kept_rows_bitwise(P, name, nb):
    """test_refine.cpp:262-298 at the BASELINE shapes (bf16, multi-tile batches): rank-25% remasking re-decodes
    exactly K/4 rows per bin and returns every other row of the first pass unchanged."""
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, nb)
    sched = P.RevealSchedule(steps=cfg.steps)
    rm = P.RemaskConfig(rank_fraction=0.25)
    base = ctx.refine(S, wl.k, sched)
    grid, tr = ctx.refine(S, wl.k, sched, rm, want_trace=True)
    mask = tr["remask_mask"].astype(bool)
    assert np.all(mask.sum(axis=1) == max(1, wl.k // 4))
    assert np.array_equal(grid[~mask], base[~mask])
    assert np.all(tr["n_passes"] == 2)
    assert np.all(tr["remask_steps"][:, 0] == max(1, cfg.steps * max(1, wl.k // 4) // wl.k))
    # and the graph-replayed product call (no trace) returns the same grids
    assert np.array_equal(ctx.refine(S, wl.k, sched, rm), grid)


def irregular_code(rng, checks, slots, q, max_deg):
    """Edges sorted by (check, slot) with check degrees 1 .. max_deg, some slots in no check at all."""
    rows = []
    free = rng.choice(slots, size=max(1, slots // 5), replace=False)  # slots without checks
    usable = np.setdiff1d(np.arange(slots), free)
    for c in range(checks):
        deg = int(rng.integers(1, max_deg + 1))
        for l in sorted(rng.choice(usable, size=min(deg, usable.size), replace=False)):
            rows.append((c, int(l), int(rng.integers(1, q))))
    return np.array(rows, np.int32), free


@pytest.mark.parametrize("m,dim,hidden,heads,k", [(6, 128, 256, 4, 3), (8, 256, 512, 8, 8), (6, 128, 512, 0, 4), (6, 64, 128, 2, 5)])
def test_bf16_irregular_codes_match_the_oracle(P, oracle, m, dim, hidden, heads, k):
    """Codes that are not check-regular (degrees 1-7, slots in no check: test_denoiser.cpp:249-267's empty
    neighbourhoods) leave the fixed-degree fast paths: BF16 forward against the oracle, and zero messages on
    the unconnected slots."""
    rng = np.random.default_rng(100 + m + k)
    slots, checks, nb = 24, 9, 5
    model = P.Model(m=m, dim=dim, hidden=hidden, layers=2, heads=heads, precision=P.BF16)
    edges, free = irregular_code(rng, checks, slots, model.q, 7)
    w = P.weights_init(model, 3)
    ctx = P.Context(model, w, edges, checks, slots)
    S = np.log(rng.dirichlet(np.ones(model.q), size=(nb, slots))).astype(np.float32)
    X = rng.integers(0, model.q, size=(nb, k, slots))
    X = np.where(rng.random(X.shape) < 0.5, -1, X).astype(np.int32)
    lg, inc = ctx.denoise(X, S, want_incoming=True)
    wr = P.model_weights_as_run(model, w)
    for b in (0, nb - 1):
        lo, io = oracle.denoise(model, wr, edges, checks, slots, X[b], S[b].astype(np.float64), True)
        el = np.abs(lg[b] - lo).max() / np.abs(lo).max()
        ei = np.abs(inc[b] - io).max() / max(1e-30, np.abs(io).max())
        print(f"irregular m={m} D={dim} K={k} heads={heads}: logits {el:.2e} messages {ei:.2e}")
        assert el < 1e-2 and ei < 1e-2, (el, ei)
    assert np.all(inc[:, :, :, free, :] == 0.0)
    # the refinement loop on the same code: valid symbols, deterministic
    g = ctx.refine(S, k, P.RevealSchedule(steps=4), P.RemaskConfig(rank_fraction=0.25))
    assert np.all((g >= 0) & (g < model.q)) and np.array_equal(g, ctx.refine(S, k, P.RevealSchedule(steps=4), P.RemaskConfig(rank_fraction=0.25)))


def test_concurrent_calls_on_one_context_are_safe(P):
    """The reference calls Denoiser::logits concurrently from its parallel_for workers on one shared instance
    (uradec.cpp:184, 294-297): 8 host threads mixing cider_denoise and cider_refine on ONE context (ctypes
    drops the GIL) must each get what the serial call returns."""
    import threading
    cfg = P.configs()["c2"]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    sched, rm = P.RevealSchedule(steps=cfg.steps), P.RemaskConfig(rank_fraction=0.25)
    jobs = []
    for t in range(8):
        nb = 3 + 5 * t
        _, S = wl.bins(e, 100 * t, nb)
        X = np.full((nb, wl.k, wl.slots), -1, np.int32)
        X[:, t % wl.k, ::3] = t
        jobs.append((S, X))
    serial = [(ctx.denoise(X, S), ctx.refine(S, wl.k, sched, rm)) for S, X in jobs]
    out = [None] * len(jobs)
    errs = []

    def work(i):
        try:
            S, X = jobs[i]
            for _ in range(3):
                out[i] = (ctx.denoise(X, S), ctx.refine(S, wl.k, sched, rm))
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs
    for (lg, g), (lg2, g2) in zip(serial, out):
        assert np.array_equal(lg, lg2) and np.array_equal(g, g2)


def _sweep_cases():
    """Seeded random small configurations of the whole loop (FP32 parity mode): field size, users, slots,
    checks, layers, heads (0 = the reference's plain extrinsic mean), schedule shape, remask mode."""
    rng = np.random.default_rng(2605)
    cases = []
    for i in range(14):
        m = int(rng.choice([2, 3, 4, 5, 6]))
        dim = int(rng.choice([16, 32, 48]))
        heads = int(rng.choice([0, 1, 2, 4]))
        hidden = int(rng.choice([dim, 2 * dim, 24]))
        layers = int(rng.integers(1, 4))
        k = int(rng.integers(1, 7))
        slots = int(rng.choice([6, 9, 12, 20]))
        checks = int(rng.integers(3, max(4, slots // 2 + 1)))
        steps = int(rng.integers(1, 9))
        tau = [(1.0, 1.0), (2.0, 0.5), (1.5, 0.2)][int(rng.integers(0, 3))]
        first = bool(rng.integers(0, 2))
        rmode = int(rng.integers(0, 3))
        cases.append((i, m, dim, hidden, layers, heads, k, slots, checks, steps, tau, first, rmode))
    # widths that are no multiple of anything (the reference takes any dim: denoiser.cpp:41-44)
    cases += [(14, 3, 10, 7, 1, 5, 2, 6, 3, 3, (1.0, 1.0), True, 0), (15, 2, 1, 1, 1, 0, 2, 6, 3, 2, (1.0, 1.0), True, 1),
              (16, 4, 33, 33, 2, 3, 3, 9, 4, 4, (1.5, 0.2), False, 2), (17, 1, 3, 5, 2, 1, 2, 8, 4, 3, (1.0, 1.0), True, 1),
              # more steps than sites (most steps reveal nothing; with K = 1 the first reveal takes every site)
              (18, 3, 16, 16, 1, 0, 1, 6, 3, 40, (1.0, 1.0), True, 1), (19, 3, 16, 16, 1, 2, 2, 6, 3, 40, (2.0, 0.5), False, 2),
              (20, 4, 16, 16, 1, 0, 6, 6, 3, 64, (1.0, 1.0), True, 2)]
    return cases


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"s{c[0]}-m{c[1]}-K{c[6]}-L{c[7]}-T{c[9]}-r{c[12]}")
def test_fp32_random_configurations_decode_like_the_oracle(P, oracle, case):
    """Identical grids, first-reveal counts and remask rows / steps / masks against the oracle for seeded random
    shapes and schedules — the loop logic (reveal targets, ties, residual forcing, threshold buckets, rank
    selection) is shared by both precision modes."""
    i, m, dim, hidden, layers, heads, k, slots, checks, steps, tau, first, rmode = case
    wl = P.Workload(m=m, slots=slots, checks=checks, k=k, snr_db=3.0, p_erase=0.15, p_false=0.15)
    model = P.Model(m=m, dim=dim, hidden=hidden, layers=layers, heads=heads, precision=P.FP32)
    e = wl.code()
    w = P.weights_init(model, 10 + i)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    ctx.set_debug_guard(65536)
    nb = 5
    _, S = wl.bins(e, 7 * i, nb)
    sched = P.RevealSchedule(steps=steps, tau_max=tau[0], tau_min=tau[1], first_reveal=first)
    rm = [None, P.RemaskConfig(rank_fraction=0.34), P.RemaskConfig(thresholds=(0.9, 0.5))][rmode]
    grid, tr = ctx.refine(S, k, sched, rm, want_trace=True)
    ro = oracle.refine(model, P.model_weights_as_run(model, w), e, wl.checks, wl.slots, S.astype(np.float64), k, sched, rm)
    assert np.array_equal(grid, ro["grid"])
    assert np.array_equal(tr["first_reveals"], ro["first_reveals"])
    assert np.array_equal(tr["remask_rows"], ro["remask_rows"])
    assert np.array_equal(tr["remask_steps"], ro["remask_steps"])
    assert np.array_equal(tr["remask_mask"], ro["remask_mask"])
    assert np.array_equal(ctx.refine(S, k, sched, rm), grid)  # the graph-replayed call
    bad, msg = ctx.debug_check()
    assert bad == 0, msg


def _bf16_sweep_cases():
    rng = np.random.default_rng(26580)
    cases = []
    for i in range(12):
        m = int(rng.choice([6, 7, 8]))
        dim = int(rng.choice([64, 128, 256]))
        hidden = int(rng.choice([64, 128, 256, 512]))
        heads = int(rng.choice([0, 1, 2, 4, 8]))
        layers = int(rng.integers(1, 4))
        k = int(rng.integers(1, 9))
        slots = int(rng.choice([8, 12, 16, 24, 40]))
        checks = int(rng.integers(3, slots // 2 + 1))
        nb = int(rng.choice([1, 3, 17, 33]))
        cases.append((i, m, dim, hidden, layers, heads, k, slots, checks, nb))
    # many users per bin (K up to the ABI's 32), a long code, a wide hidden layer, a batch of several row tiles
    cases += [(12, 8, 256, 1024, 1, 8, 16, 12, 6, 9), (13, 8, 256, 256, 2, 8, 32, 8, 4, 5), (14, 6, 128, 512, 1, 8, 4, 200, 100, 40),
              (15, 8, 256, 1024, 2, 8, 8, 64, 32, 70), (16, 7, 128, 256, 1, 4, 32, 16, 8, 3)]
    return cases


@pytest.mark.parametrize("case", _bf16_sweep_cases(), ids=lambda c: f"b{c[0]}-m{c[1]}-D{c[2]}-H{c[3]}-h{c[5]}-K{c[6]}-L{c[7]}-P{c[8]}-B{c[9]}")
def test_bf16_random_configurations_match_the_oracle(P, oracle, case):
    """Seeded random BF16 shapes (the dispatcher mixes the 2-SM fused kernels, the 1-SM ones and the generic
    kernels depending on Q, D, H, K, the check degrees and the batch): forward logits and per-layer messages
    within 1e-2 of the oracle on the first and last bin; the refinement returns valid symbols, deterministically,
    independent of the internal chunking."""
    i, m, dim, hidden, layers, heads, k, slots, checks, nb = case
    wl = P.Workload(m=m, slots=slots, checks=checks, k=k, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=m, dim=dim, hidden=hidden, layers=layers, heads=heads, precision=P.BF16)
    e = wl.code()
    w = P.weights_init(model, 20 + i)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    ctx.set_debug_guard(65536)  # 0xA5 bands around every workspace buffer: no kernel may write past its rows
    _, S = wl.bins(e, 3 * i, nb)
    rng = np.random.default_rng(i)
    X = rng.integers(0, model.q, size=(nb, k, slots))
    X = np.where(rng.random(X.shape) < 0.5, -1, X).astype(np.int32)
    lg, inc = ctx.denoise(X, S, want_incoming=True)
    wr = P.model_weights_as_run(model, w)
    for b in sorted({0, nb - 1}):
        lo, io = oracle.denoise(model, wr, e, wl.checks, wl.slots, X[b], S[b].astype(np.float64), True)
        el = np.abs(lg[b] - lo).max() / np.abs(lo).max()
        ei = np.abs(inc[b] - io).max() / max(1e-30, np.abs(io).max())
        print(f"bf16 sweep {case}: logits {el:.2e} messages {ei:.2e}")
        assert el < 1e-2 and ei < 1e-2, (case, el, ei)
    sched = P.RevealSchedule(steps=3)
    rm = P.RemaskConfig(rank_fraction=0.25)
    g = ctx.refine(S, k, sched, rm)
    assert np.all((g >= 0) & (g < model.q))
    ctx.set_chunk(max(1, nb // 2))
    assert np.array_equal(ctx.refine(S, k, sched, rm), g)
    ctx.refine(S, k, sched, P.RemaskConfig(thresholds=(0.9, 0.3)), want_trace=True)
    bad, msg = ctx.debug_check()
    assert bad == 0, msg


def _bp_sweep_cases():
    rng = np.random.default_rng(7)
    cases = []
    for i in range(10):
        m = int(rng.choice([2, 3, 4, 5, 6, 8]))
        slots = int(rng.choice([6, 9, 12, 20, 33]))
        checks = int(rng.integers(3, slots // 2 + 1))
        k = int(rng.integers(1, 5))
        nb = int(rng.choice([1, 5, 19]))
        iters = int(rng.choice([1, 7, 25]))
        cases.append((i, m, slots, checks, k, nb, iters))
    return cases


@pytest.mark.parametrize("case", _bp_sweep_cases(), ids=lambda c: f"bp{c[0]}-m{c[1]}-L{c[2]}-P{c[3]}-K{c[4]}-B{c[5]}-it{c[6]}")
def test_bp_random_configurations_match_the_reference(P, reference, case):
    """SURVEY §8(f) F1 on seeded random shapes (dense and sparse checks, Q = 4 .. 256): bp_decode and sic_decode
    against the compiled reference — identical hard decisions, flags, iteration counts and SIC grids."""
    i, m, slots, checks, k, nb, iters = case
    wl = P.Workload(m=m, slots=slots, checks=checks, k=k, snr_db=6.0, p_erase=0.05, p_false=0.05)
    e = wl.code()
    _, S = wl.bins(e, 11 * i, nb)
    S = S.astype(np.float64)
    lam = np.exp(S - S.max(axis=-1, keepdims=True))
    lam /= lam.sum(axis=-1, keepdims=True)
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    cfg = P.BpConfig(max_iters=iters)
    hard, marg, conv, its = dec.bp_decode(lam, cfg)
    rh, rm, rc, ri = reference.bp_decode(wl.m, e, wl.checks, wl.slots, lam, max_iters=iters)
    assert np.array_equal(hard, rh)
    assert np.array_equal(conv, rc.astype(bool))
    assert np.array_equal(its, ri)
    assert np.abs(marg - rm).max() / np.abs(rm).max() < 1e-9
    grid, sc, si = dec.sic_decode(S, wl.k, cfg)
    rg, rsc, rsi = reference.sic_decode(wl.m, e, wl.checks, wl.slots, S, wl.k, max_iters=iters)
    assert np.array_equal(grid, rg)
    assert np.array_equal(sc, rsc.astype(bool))
    assert np.array_equal(si, rsi)


@pytest.mark.parametrize("m,d", [(1, 2), (2, 3), (3, 7), (5, 2), (5, 9), (7, 4), (8, 12), (8, 2), (4, 16)])
def test_wht_check_update_sweep(P, oracle, m, d):
    """SURVEY §8(a) A14 over field sizes 2..256 and check degrees 2..16 (test_bp.cpp:145-168 runs degree 3
    only): the device's shuffle-butterfly WHT update against the oracle's restatement of check_update_wht,
    peaked and flat messages alike."""
    q = 1 << m
    rng = np.random.default_rng(1000 + 17 * m + d)
    n = 37
    v2c = rng.random((n, d, q)) ** rng.choice([1, 3, 8], size=(n, d, 1))
    v2c /= v2c.sum(-1, keepdims=True)
    cf = rng.integers(1, q, size=(n, d)).astype(np.int32)
    out = P.check_update_wht(m, v2c, cf)
    assert out.shape == (n, d, q) and np.allclose(out.sum(-1), 1.0)
    for c in (0, 11, n - 1):
        for i in range(d):
            others = [j for j in range(d) if j != i]
            ref = oracle.check_update_wht(m, v2c[c, others], cf[c, others], int(cf[c, i]))
            assert np.abs(out[c, i] - ref).max() < 1e-8


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_degenerate_inputs_return_errors_or_empty_results(P, oracle, prec):
    """Boundary inputs through the C ABI: no bins, no rows, too many rows, bad tokens, an edgeless code
    (test_denoiser.cpp:249-267: Module B reduces to nothing), a single slot per check — errors come back as the
    reference's exception types (status 3 -> ValueError), never as a crash, and the context stays usable."""
    bf = prec == "bf16"
    m, dim, hid = (6, 64, 128) if bf else (3, 16, 16)
    model = P.Model(m=m, dim=dim, hidden=hid, layers=2, heads=2, precision=P.BF16 if bf else P.FP32)
    wl = P.Workload(m=m, slots=10, checks=4, k=3, snr_db=5.0)
    e = wl.code()
    w = P.weights_init(model, 4)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 2)
    q = model.q
    sched = P.RevealSchedule(steps=3)
    assert ctx.denoise(np.zeros((0, 3, 10), np.int32), S[:0]).shape == (0, 3, 10, q)
    assert ctx.refine(S[:0], 3, sched).shape == (0, 3, 10)
    for bad in (q, q + 100, -2, -(1 << 30)):
        X = np.zeros((2, 3, 10), np.int32)
        X[1, 2, 9] = bad
        with pytest.raises(ValueError, match="token out of range"):
            ctx.denoise(X, S)
    with pytest.raises(ValueError):
        ctx.refine(S, 0, sched)
    with pytest.raises(ValueError):
        ctx.refine(S, 33, sched)
    with pytest.raises(ValueError):
        ctx.refine(S, 3, sched, P.RemaskConfig(rank_fraction=1.5))
    good = ctx.refine(S, 3, sched)  # still usable after the failures
    assert np.all((good >= 0) & (good < q))
    # an edgeless code: no messages, the forward equals the oracle's
    none = np.zeros((0, 3), np.int32)
    ctx0 = P.Context(model, w, none, 2, 10)
    X = np.full((2, 3, 10), -1, np.int32)
    X[0, 1, 4] = 1
    lg, inc = ctx0.denoise(X, S, want_incoming=True)
    assert np.all(inc == 0.0)
    lo = oracle.denoise(model, P.model_weights_as_run(model, w), none, 2, 10, X[0], S[0].astype(np.float64))
    assert np.abs(lg[0] - lo).max() / np.abs(lo).max() < (1e-2 if bf else 1e-4)
    g0 = ctx0.refine(S, 3, sched, P.RemaskConfig(rank_fraction=0.34))
    assert np.all((g0 >= 0) & (g0 < q))
    # degree-1 checks only (every edge alone in its check: the extrinsic set of each edge is empty)
    lone = np.array([[0, 2, 1], [1, 5, q - 1], [2, 7, 3]], np.int32)
    ctx1 = P.Context(model, w, lone, 3, 10)
    lg1, inc1 = ctx1.denoise(X, S, want_incoming=True)
    lo1, io1 = oracle.denoise(model, P.model_weights_as_run(model, w), lone, 3, 10, X[0], S[0].astype(np.float64), True)
    assert np.abs(lg1[0] - lo1).max() / np.abs(lo1).max() < (1e-2 if bf else 1e-4)
    assert np.abs(inc1[0] - io1).max() <= (1e-2 if bf else 1e-4) * max(1e-30, np.abs(io1).max()) + 1e-12


def test_graph_cache_never_replays_a_stale_capture(P):
    """Refinement chunks are captured into CUDA graphs keyed by (bins, K, schedule, remask, buffers): a shuffled
    sequence of calls with different batch sizes, row counts, schedules, remask modes and final-logits requests,
    each repeated (so later calls replay), must return what a fresh context computes for that call."""
    cfg = P.configs()["c2"]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    w = P.weights_init(model, 1)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 96)
    calls = []
    for nb in (96, 17, 64):
        for k in (4, 2):
            for steps, tau in ((8, (1.0, 1.0)), (3, (2.0, 0.5))):
                for rm in (None, P.RemaskConfig(rank_fraction=0.25), P.RemaskConfig(rank_fraction=0.5)):
                    calls.append((nb, k, steps, tau, rm))
    rng = np.random.default_rng(3)
    order = list(rng.permutation(len(calls))[:14])
    order = order + order[::-1] + order
    want = {}
    for n, ci in enumerate(order):
        nb, k, steps, tau, rm = calls[ci]
        sched = P.RevealSchedule(steps=steps, tau_max=tau[0], tau_min=tau[1])
        fl_req = (n % 3 == 1)
        out = ctx.refine(S[:nb], k, sched, rm, want_final_logits=fl_req)
        grid, fl = out if fl_req else (out, None)
        if ci not in want:
            fresh = P.Context(model, w, e, wl.checks, wl.slots)
            want[ci] = fresh.refine(S[:nb], k, sched, rm, want_final_logits=True)
            fresh.close()
        assert np.array_equal(grid, want[ci][0]), (n, calls[ci])
        if fl_req:
            assert np.array_equal(fl, want[ci][1]), (n, calls[ci])


def test_bf16_ragged_loads_equal_per_load_calls(P):
    """cider_refine_ragged at the c3 model shapes in BF16: bins of 1..8 users bucketed by load, each bucket with
    its own schedule / remask — every bin's grid equals the uniform-K call on that bin alone."""
    cfg = P.configs()["c3"]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    rng = np.random.default_rng(8)
    nb = 40
    loads = rng.integers(1, 9, size=nb).astype(np.int32)
    _, S = wl.bins(e, 0, nb)
    scheds = [P.RevealSchedule(steps=2 + (k % 3)) for k in range(8)]
    rms = [None, P.RemaskConfig(rank_fraction=0.5), None, P.RemaskConfig(rank_fraction=0.25), None,
           P.RemaskConfig(thresholds=[0.02]), None, P.RemaskConfig(rank_fraction=0.25)]
    grids = ctx.refine_ragged(S, loads, scheds, rms)
    for b in range(nb):
        k = int(loads[b])
        ref = ctx.refine(S[b:b + 1], k, scheds[k - 1], rms[k - 1])
        assert grids[b].shape == (k, wl.slots) and np.array_equal(grids[b], ref[0]), (b, k)


def _workload_sweep():
    rng = np.random.default_rng(99)
    cases = []
    for i in range(10):
        m = int(rng.choice([1, 2, 3, 5, 6, 7, 8]))
        slots = int(rng.choice([6, 10, 17, 40]))
        checks = int(rng.integers(3 if m > 1 else 4, slots // 2 + 1))
        k = int(rng.integers(1, 9))
        pe = float(rng.choice([0.0, 0.05, 0.5, 1.0]))
        pf = float(rng.choice([0.0, 0.1, 1.0]))
        snr = float(rng.choice([-3.0, 4.0, 20.0]))
        first = int(rng.choice([0, 5, 100000, 262143]))
        n = int(rng.choice([1, 7, 40]))
        seed = int(rng.choice([0, 1, 12345678901]))
        cases.append((i, m, slots, checks, k, pe, pf, snr, first, n, seed))
    return cases


@pytest.mark.parametrize("case", _workload_sweep(), ids=lambda c: f"w{c[0]}-m{c[1]}-L{c[2]}-P{c[3]}-K{c[4]}-pe{c[5]}-pf{c[6]}")
def test_device_workload_sweep(P, case):
    """the device evidence generator (mt19937_64 and the libstdc++ uniform / normal / integer
    distributions restated per bin) against the host generator over field sizes 2..256, erasure and
    false-candidate probabilities 0..1, high bin indices and master seeds: identical codewords, S equal up to the
    last ulp of exp / log."""
    i, m, slots, checks, k, pe, pf, snr, first, n, seed = case
    q = 1 << m
    if k > q ** (slots - checks):  # K distinct codewords must exist
        k = 1
    wl = P.Workload(m=m, slots=slots, checks=checks, k=k, snr_db=snr, p_erase=pe, p_false=pf, master_seed=seed)
    e = wl.code()
    model = P.Model(m=m, dim=16, hidden=16, precision=P.FP32)
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    th, Sh = wl.bins(e, first, n)
    td, Sd = wl.bins_device(ctx, e, first, n)
    assert np.array_equal(th, td)
    assert np.isfinite(Sd).all()
    assert (Sd != Sh).mean() < 1e-3
    assert np.all(np.abs(Sd - Sh) <= np.spacing(np.abs(Sh)) * 1.0001)


@pytest.mark.parametrize("seed", range(6))
def test_remask_pass_sweep(P, oracle, seed):
    """ura::remask_pass with caller confidences (refine.hpp:97-100) over random shapes, confidences and thresholds,
    including thresholds no row / every row falls under and arbitrary (not decoder-produced) input grids: identical
    grids to the oracle, untouched bins bit for bit."""
    rng = np.random.default_rng(500 + seed)
    m = int(rng.choice([3, 4, 6]))
    k = int(rng.integers(1, 7))
    slots = int(rng.choice([6, 12, 16]))
    checks = int(rng.integers(3, slots // 2 + 1))
    model = P.Model(m=m, dim=int(rng.choice([16, 32, 64])), hidden=32, layers=int(rng.integers(1, 3)),
                    heads=int(rng.choice([0, 2])), precision=P.FP32)
    wl = P.Workload(m=m, slots=slots, checks=checks, k=k, snr_db=4.0, p_erase=0.1, p_false=0.1)
    e = wl.code()
    w = P.weights_init(model, 30 + seed)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    nb = 7
    _, S = wl.bins(e, seed, nb)
    sched = P.RevealSchedule(steps=int(rng.integers(1, 9)), tau_max=1.5, tau_min=0.5, first_reveal=bool(rng.integers(0, 2)))
    g0 = rng.integers(0, model.q, size=(nb, k, slots)).astype(np.int32)
    conf = rng.random((nb, k))
    wr = P.model_weights_as_run(model, w)
    for thr in (0.0, 0.35, 0.7, 1.01):
        g = ctx.remask_pass(S, g0, conf, thr, sched)
        go, _ = oracle.remask_pass(model, wr, e, wl.checks, wl.slots, S.astype(np.float64), g0, conf, thr, sched)
        assert np.array_equal(g, go), (seed, thr)
        keep = ~(conf < thr)
        assert np.array_equal(g[keep], g0[keep])
