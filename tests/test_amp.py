"""the batched AMP slot detector (the evidence the refinement path consumes).

The device detector (`AmpDetector`, C ABI `cider_amp_*`) against the reference's own detect_frame
(amp.cpp:133-148, compiled in oracle/_ref) on frames the reference itself generates
(make_dictionaries + activity_vector + transmit, sim.cpp). Both compute in fp64 in the same operation
order; they differ only through the libm exp / log / log1p of the two platforms (<= 1 ulp), so the
evidence rows agree to 1e-8 absolute (entries are natural logs in [-40, 0]) and the per-slot
ranking of the symbols is identical.
"""
import numpy as np
import pytest

from oracle.binding import have_reference


def frames(ref, q, n_s, slots, k, B, eb_db=10.0, seed=7):
    dicts = ref.amp_make_dicts(q, n_s, slots, seed)
    p_sym = ref.symbol_power(eb_db, 24, slots)
    rng = np.random.default_rng(seed)
    sym = rng.integers(0, q, size=(B, slots, k)).astype(np.int32)
    y = np.stack([ref.amp_observe(dicts, sym[b], p_sym, 1.0, 1000 + b) for b in range(B)])
    return dicts, y, p_sym, sym


@pytest.mark.skipif(not have_reference(), reason="needs oracle/_ref (reference sources)")
def test_reference_amp_shim_runs():
    from oracle.binding import Reference
    ref = Reference()
    dicts, y, p_sym, sym = frames(ref, 64, 24, 12, 2, 2)
    S = ref.amp_detect_frame(dicts, y[0], 20, 2 / 64, p_sym, -40.0)
    assert S.shape == (12, 64) and np.all(S <= 0.0) and np.all(S >= -40.0)
    # the transmitted symbols carry the most evidence in (almost) every slot
    top2 = np.argsort(-S, axis=1)[:, :2]
    hits = np.mean([set(sym[0, l]) <= set(top2[l]) for l in range(12)])
    assert hits > 0.5


@pytest.mark.gpu
@pytest.mark.parametrize("q,n_s,slots,k,B", [(64, 24, 12, 2, 16), (256, 64, 16, 4, 6)])
def test_amp_detect_matches_reference(P, q, n_s, slots, k, B):
    if not have_reference():
        pytest.skip("needs oracle/_ref")
    from oracle.binding import Reference
    ref = Reference()
    dicts, y, p_sym, _ = frames(ref, q, n_s, slots, k, B)
    cfg = P.AmpConfig(iters=20, rho_bg=k / q, sigma_u2=p_sym, evidence_floor=-40.0)
    det = P.AmpDetector(dicts)
    S = det.detect(y, cfg)
    for b in range(B):
        R = ref.amp_detect_frame(dicts, y[b], cfg.iters, cfg.rho_bg, cfg.sigma_u2, cfg.evidence_floor)
        assert np.abs(S[b] - R).max() < 1e-8
        assert np.array_equal(np.argsort(-S[b], axis=1, kind="stable")[:, :k], np.argsort(-R, axis=1, kind="stable")[:, :k])


@pytest.mark.gpu
def test_amp_errors_like_the_reference(P):
    dicts = np.exp(1j * np.random.default_rng(0).random((2, 8, 4)))
    det = P.AmpDetector(dicts)
    y = np.zeros((1, 2, 4), np.complex128)
    with pytest.raises(ValueError, match="need at least one iteration"):
        det.detect(y, P.AmpConfig(iters=0))
    with pytest.raises(ValueError, match="rho_bg must lie in"):
        det.detect(y, P.AmpConfig(rho_bg=1.5))
    with pytest.raises(ValueError, match="sigma_u2 must be positive"):
        det.detect(y, P.AmpConfig(sigma_u2=0.0))
    with pytest.raises(ValueError, match="n_s must not exceed Q"):
        P.AmpDetector(np.ones((1, 4, 8), np.complex128))
    assert det.detect(y[:0]).shape == (0, 2, 8)


def _amp_sweep():
    rng = np.random.default_rng(11)
    cases = []
    for i in range(8):
        q = int(rng.choice([4, 16, 32, 64, 128, 256]))
        n_s = int(rng.integers(2, q + 1))
        slots = int(rng.choice([1, 3, 8, 20]))
        k = int(rng.integers(1, min(q, 6) + 1))
        B = int(rng.choice([1, 4, 9]))
        iters = int(rng.choice([1, 5, 20]))
        cases.append((i, q, n_s, slots, k, B, iters))
    return cases


@pytest.mark.gpu
@pytest.mark.parametrize("case", _amp_sweep(), ids=lambda c: f"amp{c[0]}-q{c[1]}-ns{c[2]}-L{c[3]}-K{c[4]}-B{c[5]}-it{c[6]}")
def test_amp_random_configurations_match_reference(P, case):
    """Seeded random detector shapes (Q = 4..256, n_s from 2 to Q, one slot to twenty, one to twenty iterations)."""
    if not have_reference():
        pytest.skip("needs oracle/_ref")
    from oracle.binding import Reference
    ref = Reference()
    i, q, n_s, slots, k, B, iters = case
    dicts, y, p_sym, _ = frames(ref, q, n_s, slots, k, B, seed=20 + i)
    cfg = P.AmpConfig(iters=iters, rho_bg=min(0.9, k / q), sigma_u2=p_sym, evidence_floor=-40.0)
    S = P.AmpDetector(dicts).detect(y, cfg)
    for b in range(B):
        R = ref.amp_detect_frame(dicts, y[b], cfg.iters, cfg.rho_bg, cfg.sigma_u2, cfg.evidence_floor)
        assert np.abs(S[b] - R).max() < 1e-8, np.abs(S[b] - R).max()
