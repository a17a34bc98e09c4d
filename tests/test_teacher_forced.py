"""CPU checks of the teacher-forced decision checker (tests/teacher_forced.py) on the oracle's own
trajectories: the oracle's record stream reproduces oracle.refine, checks clean against itself, and
the checker tells a near-tie flip (explained) from a real one (unexplained)."""
import numpy as np

from oracle import teacher_forced as tf


def _case(P):
    wl = P.Workload(m=4, slots=12, checks=6, k=4, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=4, dim=24, hidden=32, layers=2, heads=2)
    e = wl.code()
    w = P.weights_init(model, 3).astype(np.float64)
    _, S = wl.bins(e, 0, 2)
    return wl, model, e, w, S


def test_oracle_trajectory_matches_refine(P, oracle):
    wl, model, e, w, S = _case(P)
    sched = P.RevealSchedule(steps=5)
    rm = P.RemaskConfig(rank_fraction=0.5)
    for b in range(2):
        meta, X, lg, g = tf.oracle_trajectory(oracle, model, w, e, wl, S[b], sched, k_low=2)
        ro = oracle.refine(model, w, e, wl.checks, wl.slots, S[b:b + 1].astype(np.float64), wl.k, sched, rm)
        assert np.array_equal(g, ro["grid"][0])
        assert meta.shape[0] == (5 + 2) + (2 + 2)  # pass 0: 5 steps + final + output; pass 1: T_rm=2 ...
        st = tf.check_bin(tf.Stats(), b, meta, X, lg, lg, sched, 2)
        assert st.flips == 0 and not st.unexplained and st.carry_mismatch == 0 and st.decisions > 0


def test_checker_explains_near_ties_only(P, oracle):
    wl, model, e, w, S = _case(P)
    sched = P.RevealSchedule(steps=5)
    meta, X, lg, _ = tf.oracle_trajectory(oracle, model, w, e, wl, S[0], sched, k_low=0)
    # a value flip at the last step's final pass where the oracle margin is large -> unexplained
    r = int(np.nonzero(meta[:, 3] == 1)[0][0])
    Xb = X.copy()
    top2 = np.sort(lg[r], -1)[..., -2:]
    gap = top2[..., 1] - top2[..., 0]
    k, l = np.unravel_index(np.argmax(gap), gap.shape)
    second = int(np.argsort(lg[r][k, l])[-2])
    Xb[r + 1][k, l] = second
    st = tf.check_bin(tf.Stats(), 0, meta, Xb, lg, lg, sched, 0)
    assert st.flips == 1 and len(st.unexplained) == 1
    # the same flip with a device logit error larger than the gap -> explained
    lgd = lg.copy()
    lgd[r][k, l, second] += gap[k, l] * 0.6
    lgd[r][k, l, int(np.argmax(lg[r][k, l]))] -= gap[k, l] * 0.6
    st = tf.check_bin(tf.Stats(), 0, meta, Xb, lgd, lg, sched, 0)
    assert st.flips == 1 and st.explained == 1 and not st.unexplained
