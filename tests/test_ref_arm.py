"""The reference arm's inputs and engine (bench.py --impl reference): the shim's weight init and
evidence generator reproduce the product's host generators bit for bit (so both arms decode the same
bins with the same weights), and the paused-between-forwards session is the reference's own decode."""
import numpy as np
import pytest


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_ref_inputs_equal_product_inputs(P, reference, name):
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    from oracle.binding import derive_seed
    e_ref = reference.build_ldpc(wl.m, wl.slots, wl.checks, wl.col_weight, derive_seed(0, 1))
    e = wl.code()
    assert np.array_equal(e_ref, e)
    t_ref, S_ref = reference.workload_bins(wl, e_ref, 5, 3)
    t, S = wl.bins(e, 5, 3)
    assert np.array_equal(t_ref, t) and np.array_equal(S_ref, S.astype(np.float64))
    w_ref = reference.weights_init(model, 1)
    assert np.array_equal(w_ref, P.weights_init(model, 1, f64=True))


def test_ref_weights_init_is_random_init_in_ref_exact_mode(P, reference):
    m = P.Model.ref_exact(4, 16)
    assert np.array_equal(reference.weights_init(m, 9), reference.random_init(16, 16, 9))


def test_ref_session_decodes_like_ref_refine(P, reference):
    from oracle.binding import RefSession
    wl = P.Workload(m=4, slots=12, checks=6, k=4, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=4, dim=16, hidden=24, layers=2, heads=2)
    e = wl.code()
    w = reference.weights_init(model, 2)
    _, S = reference.workload_bins(wl, e, 0, 5)
    sched = P.RevealSchedule(steps=4)
    rm = P.RemaskConfig(rank_fraction=0.5)
    ses = RefSession(reference, model, w, e, wl.checks, wl.slots, wl.k, S, sched, rm, threads=2)
    per_bin = P.forward_count(P.Config("x", wl, model, 5, 4, rm))
    st0 = ses.status()
    assert st0["forwards"] == 0
    ses.advance(1)
    assert ses.status()["forwards"] == 2
    for _ in range(3 * per_bin):
        ses.advance(1)
    st = ses.status()
    ses.close()
    assert st["done"].all() and st["bins_done"] == 5 and st["forwards"] == 5 * per_bin
    ro = reference.refine(model, w, e, wl.checks, wl.slots, S, wl.k, sched, rm)
    assert np.array_equal(st["grids"], ro["grid"])
