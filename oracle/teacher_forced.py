"""Teacher-forced, margin-aware decision checker — TEST INFRASTRUCTURE ONLY
(used by tests/ and bench.py's parity leg as the checker, never on the measured path).

The device decodes a batch through `cider_refine_probe`, which records, for a few probe bins, every
denoiser forward's input grid X_r and output logits, and every pass's output grid (execution order).
For each record the CPU oracle is fed the SAME input grid (teacher forcing on the device's own
trajectory, so no divergence accumulates) and every device decision is re-derived from the oracle's
logits with the reference's rules:

  reveal_step     refine.cpp:83-127   (first step: one site per slot, strict >, lowest row;
                                       else (kappa desc, row asc, slot asc) until the cosine target)
  residual force  refine.cpp:175-178
  final argmax    refine.cpp:187-192  (updatable rows only)
  rank remask     SURVEY §7.1(3) over MaxProbScorer row confidences (refine.cpp:207-225, 238-275)

A decision that differs from the oracle's is a FLIP. A flip is EXPLAINED when the oracle's own margin
for it is below what the measured logit error of that record can move it by:
  * selection flip (site / row chosen by one side only): |log kappa_a - log kappa_b| <= 4 eps / tau
    (eps = max |logit_dev - logit_oracle| over the bin; each log kappa moves by <= 2 eps / tau);
  * value flip (argmax symbol differs): oracle top-1 minus the device's symbol <= 2 eps_site;
  * remask row flip: |c_a - c_b| <= (c_a + c_b) (e^{2 eps} - 1) on MaxProb row confidences.
Every other site must be carried over bit for bit. The checker returns counts; tests assert
`unexplained == 0` and report agreement rates.
"""
from __future__ import annotations

import math

import numpy as np


def _kappa(lam: np.ndarray, tau: float) -> np.ndarray:
    """site confidence kappa = 1 / sum_a exp((lam_a - max) / tau) (refine.cpp:61-70), fp64."""
    m = lam.max(-1, keepdims=True)
    return 1.0 / np.exp((lam - m) / tau).sum(-1)


def _cosfrac(t: int, T: int) -> float:
    return 0.5 * (1.0 - math.cos(math.pi * t / T))


def _temperature(t: int, T: int, tmax: float, tmin: float) -> float:
    if T <= 1:
        return tmin
    w = 0.5 * (1.0 + math.cos(math.pi * (t - 1) / (T - 1)))
    return tmax * w + tmin * (1.0 - w)


def _lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


class Stats:
    def __init__(self):
        self.decisions = 0          # site / row decisions compared
        self.flips = 0              # decisions that differ from the oracle's
        self.explained = 0          # flips within the measured error margin
        self.unexplained = []       # (bin, record, what, detail)
        self.max_rel_err = 0.0      # max over records of max|dev - oracle| / max|oracle|
        self.carry_mismatch = 0     # non-decision sites that changed (must be 0)
        self.records = 0

    @property
    def agreement(self) -> float:
        return 1.0 - self.flips / max(1, self.decisions)

    def as_dict(self) -> dict:
        return {"decisions": self.decisions, "flips": self.flips, "explained_flips": self.explained,
                "unexplained_flips": len(self.unexplained), "decision_agreement": round(self.agreement, 6),
                "max_logit_rel_err": float(self.max_rel_err), "records": self.records,
                "carry_mismatch": self.carry_mismatch}


def check_bin(st: Stats, b: int, meta: np.ndarray, X: np.ndarray, lg_dev: np.ndarray, lg_orc: np.ndarray,
              sched, k_low: int):
    """One probe bin: meta R x 4, X R x K x L (device), lg_dev / lg_orc R x K x L x Q (kind 2 rows unused)."""
    R = meta.shape[0]
    K, L = X.shape[1:]
    pass_start = None
    upd = np.ones(K, bool)
    for r in range(R):
        p, t, T, kind = (int(v) for v in meta[r])
        if kind == 2:
            if r + 1 < R and int(meta[r + 1][3]) == 0:  # -> remask selection of the next pass
                _check_remask(st, b, r, X[r], X[r + 1], lg_dev[r - 1], lg_orc[r - 1], k_low)
                upd = np.all(X[r + 1] == -1, axis=1)
            continue
        st.records += 1
        lo, ld = lg_orc[r], lg_dev[r].astype(np.float64)
        err = np.abs(ld - lo).max(-1)  # per site
        eps = float(err.max())
        st.max_rel_err = max(st.max_rel_err, eps / max(1e-30, float(np.abs(lo).max())))
        x0, x1 = X[r], X[r + 1]
        if kind == 0:
            if t == 1:
                pass_start = x0.copy()
            init_masked = int((pass_start == -1).sum())
            base = K * L - init_masked
            tau = _temperature(t, T, sched.tau_max, sched.tau_min)
            first = t == 1 and sched.first_reveal
            masked = x0 == -1
            newly = masked & (x1 != -1)
            # carried sites must not change
            st.carry_mismatch += int((x0[~masked] != x1[~masked]).sum())
            kap = _kappa(lo, tau)
            lk = np.log(kap)
            margin = 4 * eps / tau * (1 + 1e-9) + 1e-12
            if r + 1 < R and int(meta[r + 1][3]) == 1:
                # last step: whatever the reveal leaves masked is forced to the same argmax
                # (refine.cpp:175-178), so only the values are decisions
                st.carry_mismatch += int((x1 == -1).sum())
                _check_values(st, b, r, x1, lo, err, [(int(k), int(l)) for k, l in zip(*np.nonzero(masked))])
            elif first:
                for l in range(L):
                    rows = np.nonzero(masked[:, l])[0]
                    if not len(rows):
                        continue
                    best = rows[0]
                    for k in rows[1:]:
                        if kap[k, l] > kap[best, l]:
                            best = k
                    dev = np.nonzero(newly[:, l])[0]
                    st.decisions += 1
                    if len(dev) != 1 or dev[0] != best:
                        st.flips += 1
                        ok = len(dev) == 1 and abs(lk[dev[0], l] - lk[best, l]) <= margin
                        _tally(st, ok, b, r, "first-reveal row", (l, int(best), dev.tolist()))
                    _check_values(st, b, r, x1, lo, err, [(int(k), l) for k in dev])
            else:
                target = base + _lround(_cosfrac(t, T) * init_masked)
                need = target - int((~masked).sum())
                dev = {(int(k), int(l)) for k, l in zip(*np.nonzero(newly))}
                if need > 0:
                    sites = [(int(k), int(l)) for k, l in zip(*np.nonzero(masked))]
                    sites.sort(key=lambda s_: (-kap[s_], s_[0], s_[1]))
                    orc = set(sites[:need])
                    st.decisions += len(sites)
                    plus, minus = dev - orc, orc - dev
                    if plus or minus:
                        st.flips += len(plus) + len(minus)
                        # the device ranks every site of `plus` above every site of `minus`: possible only
                        # if the oracle's log-kappa gap between the two sets is within 4 eps / tau
                        gap = (max(lk[s_] for s_ in minus) - min(lk[s_] for s_ in plus)) if plus and minus else math.inf
                        ok = len(plus) == len(minus) and gap <= margin
                        for s_ in plus | minus:
                            _tally(st, ok, b, r, "reveal set", (s_, float(lk[s_]), gap))
                else:
                    st.carry_mismatch += len(dev)
                _check_values(st, b, r, x1, lo, err, sorted(dev))
        elif kind == 1:
            # final gamma = 0 pass: updatable rows take the argmax (refine.cpp:187-192)
            rows_upd = np.nonzero(upd)[0]
            st.carry_mismatch += int((x0[~upd] != x1[~upd]).sum())
            _check_values(st, b, r, x1, lo, err, [(int(k), l) for k in rows_upd for l in range(L)])
    return st


def _check_values(st: Stats, b, r, x1, lo, err, sites):
    for (k, l) in sites:
        st.decisions += 1
        v = int(x1[k, l])
        a = int(np.argmax(lo[k, l]))  # lowest symbol on ties, as argmax_symbol
        if v == a:
            continue
        st.flips += 1
        ok = 0 <= v < lo.shape[-1] and lo[k, l, a] - lo[k, l, v] <= 2 * err[k, l] * (1 + 1e-9) + 1e-12
        _tally(st, ok, b, r, "argmax value", ((k, l), a, v, float(lo[k, l, a] - lo[k, l, v]) if 0 <= v < lo.shape[-1] else None))


def _check_remask(st: Stats, b, r, grid, x_next, lg_dev_final, lg_orc_final, k_low):
    K, L = grid.shape
    eps = float(np.abs(lg_dev_final.astype(np.float64) - lg_orc_final).max())
    conf = _kappa(lg_orc_final, 1.0).mean(-1)  # MaxProbScorer row confidence (refine.cpp:218-225)
    order = sorted(range(K), key=lambda k: (conf[k], k))
    orc = set(order[:k_low])
    dev = set(np.nonzero(np.all(x_next == -1, axis=1))[0].tolist())
    st.decisions += K
    for k in dev ^ orc:
        st.flips += 1
        other = order[k_low - 1] if k in dev else (order[k_low] if k_low < K else order[-1])
        ok = abs(conf[k] - conf[other]) <= (conf[k] + conf[other]) * (math.exp(2 * eps) - 1) * (1 + 1e-9) + 1e-15
        _tally(st, ok, b, r, "remask row", (k, float(conf[k]), float(conf[other])))
    keep = np.array([k not in dev for k in range(K)])
    st.carry_mismatch += int((grid[keep] != x_next[keep]).sum())


def _tally(st: Stats, ok: bool, b, r, what, detail):
    if ok:
        st.explained += 1
    else:
        st.unexplained.append((b, r, what, detail))


def teacher_forced(P, oracle, ctx, model, weights_run, edges, wl, S, sched, remask, probe_bins, threads=0):
    """Decode S (B bins) on the device with probes on `probe_bins`, re-run every probed forward on the
    oracle with the device's own input grids, and check all decisions. Returns (grid, Stats, details)."""
    grid, meta, X, lg = ctx.refine_probe(S, wl.k, sched, remask, probe_bins=probe_bins)
    st = Stats()
    k_low = int(math.floor(remask.rank_fraction * wl.k)) if remask is not None and remask.rank_fraction else 0
    fwd = [r for r in range(meta.shape[0]) if meta[r][3] < 2]
    n = len(probe_bins)
    Xin = np.concatenate([X[i, fwd] for i in range(n)])
    Sin = np.concatenate([np.repeat(S[b][None].astype(np.float64), len(fwd), 0) for b in probe_bins])
    lo = oracle.denoise_batch(model, weights_run, edges, wl.checks, wl.slots, Xin, Sin, threads=threads)
    lo = lo.reshape(n, len(fwd), *lo.shape[1:])
    per_bin_err = []
    for i, b in enumerate(probe_bins):
        full = np.zeros(lg.shape[1:], np.float64)
        full[fwd] = lo[i]
        check_bin(st, int(b), meta, X[i], lg[i], full, sched, k_low)
        per_bin_err.append(float(np.max([np.abs(lg[i][r] - full[r]).max() / np.abs(full[r]).max() for r in fwd])))
    return grid, st, {"meta": meta, "per_bin_rel_err": per_bin_err}


def oracle_trajectory(oracle, model, weights_run, edges, wl, S_b, sched, k_low: int = 0):
    """The oracle's own decode of one bin in cider_refine_probe's record format (meta, X, logits):
    run_masked_loop (refine.cpp:134-195) step by step through the restatement's denoise / reveal_step,
    then the rank-rule remask pass. Used to validate the checker and the probe record format."""
    K, L = wl.k, wl.slots
    metas, Xs, lgs = [], [], []

    def fwd(x):
        return oracle.denoise(model, weights_run, edges, wl.checks, wl.slots, x, S_b.astype(np.float64))

    def run_pass(p, x, T, upd):
        init_masked = int((x == -1).sum())
        base = K * L - init_masked
        lam = None
        for t in range(1, T + 1):
            lam = fwd(x)
            metas.append((p, t, T, 0)); Xs.append(x.copy()); lgs.append(lam)
            tau = _temperature(t, T, sched.tau_max, sched.tau_min)
            target = base + _lround(_cosfrac(t, T) * init_masked)
            x = oracle.reveal_step(x, lam, target, tau, t == 1 and sched.first_reveal)
        x = np.where(x == -1, lam.argmax(-1), x).astype(np.int32)
        fl = fwd(x)
        metas.append((p, 0, T, 1)); Xs.append(x.copy()); lgs.append(fl)
        out = x.copy()
        out[upd] = fl.argmax(-1)[upd]
        metas.append((p, 0, T, 2)); Xs.append(out.copy()); lgs.append(np.zeros_like(fl))
        return out, fl

    g, fl = run_pass(0, np.full((K, L), -1, np.int32), sched.steps, np.ones(K, bool))
    if k_low > 0:
        conf = _kappa(fl, 1.0).mean(-1)
        low = sorted(range(K), key=lambda k: (conf[k], k))[:k_low]
        upd = np.zeros(K, bool)
        upd[low] = True
        x0 = g.copy()
        x0[upd] = -1
        T_rm = max(1, (sched.steps * k_low) // K)
        g, _ = run_pass(1, x0, T_rm, upd)
    return np.array(metas, np.int32), np.stack(Xs), np.stack(lgs), g
