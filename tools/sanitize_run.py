"""Workload for compute-sanitizer (memcheck / synccheck / racecheck): the c3 / c5 kernel set — fused
Lambda-bar -> demix -> e (2-SM), the 2-SM gate / aggregator / fusion MLPs, the one-pass attention
pool, the CTA-pair grouped GEMMs, final logits + kappa / argmax, reveal, remask — on 40 bins of a
small degree-6 code (N=1, D=256, H=256, 8 heads), one forward and one short refinement with rank
remasking; plus the D = 128 / K = 4 variants. Prints a checksum so a run can be compared with the
unsanitised one.

  compute-sanitizer --tool memcheck  python tools/sanitize_run.py
  compute-sanitizer --tool synccheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26580_b200 as P  # noqa: E402


def run(k, dim, nb=40):
    wl = P.Workload(m=8, slots=16, checks=8, k=k, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=8, dim=dim, hidden=256, layers=1, heads=8, precision=P.BF16)
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, nb)
    rng = np.random.default_rng(5)
    X = np.where(rng.random((nb, k, wl.slots)) < 0.5, rng.integers(0, model.q, size=(nb, k, wl.slots)), -1).astype(np.int32)
    lg = ctx.denoise(X, S)
    g = ctx.refine(S, k, P.RevealSchedule(steps=3), P.RemaskConfig(rank_fraction=0.25))
    ctx.close()
    return float(np.abs(lg).sum()), int(g.sum())


if __name__ == "__main__":
    for k, dim in ((8, 256), (4, 256), (4, 128)):
        print(f"K={k} D={dim}: logits |sum| {run(k, dim)[0]:.6e}, grid sum {run(k, dim)[1]}", flush=True)
