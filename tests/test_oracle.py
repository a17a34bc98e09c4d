"""The oracle restatement against the live reference (oracle/_ref) on random cases, and the
reference's own denoiser / refine invariants (test_denoiser.cpp, test_refine.cpp) restated on it."""
import numpy as np
import pytest


def small_case(P, m=6, slots=12, checks=8, k=3, seed=0):
    wl = P.Workload(m=m, slots=slots, checks=checks, k=k, snr_db=6.0, p_erase=0.05, p_false=0.05)
    e = wl.code()
    truth, S = wl.bins(e, seed, 2)
    return wl, e, truth, S


MODELS = {
    "refexact": lambda P: P.Model.ref_exact(6, 24),
    "stacked": lambda P: P.Model(m=6, dim=32, hidden=48, layers=3),
    "attn": lambda P: P.Model(m=6, dim=32, hidden=48, layers=2, heads=4),
}


@pytest.mark.parametrize("tag", list(MODELS))
def test_denoise_bitwise_vs_reference(P, oracle, reference, tag):
    m = MODELS[tag](P)
    wl, e, _, S = small_case(P)
    w = P.weights_init(m, 5).astype(np.float64)
    rng = np.random.default_rng(1)
    for trial in range(3):
        X = rng.integers(-1, m.q, size=(3, wl.slots)).astype(np.int32)
        a, ia = oracle.denoise(m, w, e, wl.checks, wl.slots, X, S[0].astype(np.float64), True)
        b, ib = reference.denoise(m, w, e, wl.checks, wl.slots, X, S[0].astype(np.float64), True)
        assert np.array_equal(a, b) and np.array_equal(ia, ib)


@pytest.mark.parametrize("remask", [None, "thr", "rank"])
def test_refine_bitwise_vs_reference(P, oracle, reference, remask):
    m = P.Model.ref_exact(6, 16)
    wl, e, _, S = small_case(P, k=6)
    w = P.weights_init(m, 9).astype(np.float64)
    rm = {None: None, "thr": P.RemaskConfig(thresholds=(0.5, 0.2)), "rank": P.RemaskConfig(rank_fraction=0.34)}[remask]
    sched = P.RevealSchedule(steps=5, tau_max=1.7, tau_min=0.4)
    a = oracle.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 6, sched, rm, want_final_logits=True)
    b = reference.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 6, sched, rm, want_final_logits=True)
    for k in a:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k


def test_reveal_step_vs_reference(P, oracle, reference):
    rng = np.random.default_rng(4)
    for trial in range(20):
        K, L, q = rng.integers(1, 6), rng.integers(2, 14), 16
        lg = rng.normal(size=(K, L, q)).round(1)  # coarse values -> many exact ties
        X = np.where(rng.random((K, L)) < 0.3, rng.integers(0, q, size=(K, L)), -1).astype(np.int32)
        tgt = int(rng.integers(0, K * L + 1))
        tau = float(rng.uniform(0.3, 2.0))
        for first in (True, False):
            assert np.array_equal(oracle.reveal_step(X, lg, tgt, tau, first), reference.reveal_step(X, lg, tgt, tau, first))


def test_wht_vs_reference(oracle, reference):
    rng = np.random.default_rng(5)
    for m in (2, 4, 6, 8):
        q = 1 << m
        for d in (1, 2, 5):
            inc = rng.random((d, q))
            inc /= inc.sum(1, keepdims=True)
            cf = rng.integers(1, q, size=d).astype(np.int32)
            t = int(rng.integers(1, q))
            assert np.array_equal(oracle.check_update_wht(m, inc, cf, t), reference.check_update_wht(m, inc, cf, t))


# ---- the reference's invariants, restated on the oracle ---------------------------------------
def test_row_permutation_equivariance_is_exact(P, oracle):
    """test_denoiser.cpp:293-313: permuting input rows permutes the logits, bitwise."""
    m = MODELS["attn"](P)
    wl, e, _, S = small_case(P)
    w = P.weights_init(m, 2).astype(np.float64)
    X = np.random.default_rng(3).integers(-1, m.q, size=(3, wl.slots)).astype(np.int32)
    base = oracle.denoise(m, w, e, wl.checks, wl.slots, X, S[0].astype(np.float64))
    p = [2, 0, 1]
    perm = oracle.denoise(m, w, e, wl.checks, wl.slots, X[p], S[0].astype(np.float64))
    assert np.array_equal(perm, base[p])


def test_module_b_extrinsicity(P, oracle):
    """test_denoiser.cpp:213-247: changing slot l's inputs never changes slot l's own incoming
    check messages (bitwise), but does change its neighbours'."""
    m = MODELS["stacked"](P)
    wl, e, _, S = small_case(P)
    w = P.weights_init(m, 2).astype(np.float64)
    X = np.random.default_rng(8).integers(-1, m.q, size=(3, wl.slots)).astype(np.int32)
    _, base = oracle.denoise(m, w, e, wl.checks, wl.slots, X, S[0].astype(np.float64), True)
    for l in (0, 5, 11):
        Y = X.copy()
        Y[:, l] = (np.maximum(Y[:, l], 0) + 7) % m.q
        _, inc = oracle.denoise(m, w, e, wl.checks, wl.slots, Y, S[0].astype(np.float64), True)
        assert np.array_equal(inc[0][:, l], base[0][:, l])  # layer 1: extrinsic
        nbrs = {int(s) for c in e[e[:, 1] == l][:, 0] for s in e[e[:, 0] == c][:, 1]} - {l}
        assert any(not np.array_equal(inc[0][:, s], base[0][:, s]) for s in nbrs)


def test_identical_rows_tie_and_lowest_row_wins(P, oracle):
    """Identical masked rows produce identical logits (exact ties) and the first reveal picks
    the lowest row of each slot (refine.cpp:96)."""
    m = P.Model.ref_exact(6, 24)
    wl, e, _, S = small_case(P, k=4)
    w = P.weights_init(m, 2).astype(np.float64)
    X = np.full((4, wl.slots), -1, np.int32)
    lg = oracle.denoise(m, w, e, wl.checks, wl.slots, X, S[0].astype(np.float64))
    assert all(np.array_equal(lg[0], lg[k]) for k in range(1, 4))
    x1 = oracle.reveal_step(X, lg, 0, 1.0, True)
    assert np.all(x1[0] >= 0) and np.all(x1[1:] == -1)


def test_refinement_reveal_accounting_and_clamping(P, oracle):
    """First pass reveals one site per slot at t=1; remasking re-decodes only the selected rows,
    every other row stays bit-identical (refine.cpp:270-273)."""
    m = P.Model.ref_exact(6, 16)
    wl, e, _, S = small_case(P, k=6)
    w = P.weights_init(m, 4).astype(np.float64)
    sched = P.RevealSchedule(steps=6)
    plain = oracle.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 6, sched)
    assert np.all(plain["first_reveals"] == wl.slots)
    rem = oracle.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 6, sched, P.RemaskConfig(rank_fraction=0.5))
    for b in range(S.shape[0]):
        keep = rem["remask_mask"][b] == 0
        assert keep.sum() == 3 and rem["remask_rows"][b, 0] == 3 and rem["remask_steps"][b, 0] == 3
        assert np.array_equal(rem["grid"][b][keep], plain["grid"][b][keep])


def test_error_contract(P, oracle):
    m = P.Model.ref_exact(6, 16)
    wl, e, _, S = small_case(P)
    w = P.weights_init(m, 4).astype(np.float64)
    with pytest.raises(ValueError, match="embed_grid: token out of range"):
        oracle.denoise(m, w, e, wl.checks, wl.slots, np.full((2, wl.slots), 64, np.int32), S[0].astype(np.float64))
    with pytest.raises(ValueError, match="strictly descending"):
        oracle.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 3, P.RevealSchedule(steps=2),
                      P.RemaskConfig(thresholds=(0.5, 0.7)))
    with pytest.raises(ValueError, match="need T >= 1"):
        oracle.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 3, P.RevealSchedule(steps=0))


def test_oracle_threaded_forward_bitwise(P, oracle, reference):
    """The restatement's threaded forward (par_for over sites / (row, check) pairs, ordered message sums)
    and its batched entry point are bit-identical to the reference at any thread count."""
    m = P.Model(m=6, dim=32, hidden=48, layers=2, heads=4)
    wl, e, _, S = small_case(P, k=4)
    w = P.weights_init(m, 3).astype(np.float64)
    rng = np.random.default_rng(8)
    X = rng.integers(-1, m.q, size=(3, 4, wl.slots)).astype(np.int32)
    Sb = np.stack([S[0], S[1], S[0]]).astype(np.float64)
    for threads in (1, 3, 12):
        lg = oracle.denoise_batch(m, w, e, wl.checks, wl.slots, X, Sb, threads=threads)
        for b in range(3):
            assert np.array_equal(lg[b], reference.denoise(m, w, e, wl.checks, wl.slots, X[b], Sb[b]))


def test_remask_pass_with_caller_confidences_vs_reference(P, oracle, reference):
    """remask_pass on caller confidences (any ConfidenceScorer, refine.hpp:97-100): the restatement equals
    ura::remask_pass bit for bit, including bins with no low row (returned unchanged)."""
    m = P.Model(m=6, dim=24, hidden=32, layers=2, heads=2)
    wl, e, _, S = small_case(P, k=4)
    w = P.weights_init(m, 4).astype(np.float64)
    sched = P.RevealSchedule(steps=5)
    g0 = oracle.refine(m, w, e, wl.checks, wl.slots, S.astype(np.float64), 4, sched)["grid"]
    conf = np.array([[0.9, 0.1, 0.6, 0.2], [0.9, 0.8, 0.7, 0.95]])
    a, fa = oracle.remask_pass(m, w, e, wl.checks, wl.slots, S.astype(np.float64), g0, conf, 0.5, sched)
    b, fb = reference.remask_pass(m, w, e, wl.checks, wl.slots, S.astype(np.float64), g0, conf, 0.5, sched)
    assert np.array_equal(a, b) and np.array_equal(fa[0], fb[0])
    assert np.array_equal(a[1], g0[1]) and np.isnan(fa[1]).all()   # no low row: untouched
    assert np.array_equal(a[0][[0, 2]], g0[0][[0, 2]])             # clamped rows bit-identical
