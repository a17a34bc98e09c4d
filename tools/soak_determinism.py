"""Race check by repetition (compute-sanitizer is closed on the pool): the graph-replayed, PDL-chained decode of
one batch, repeated, must return bit-identical grids every time, for each BASELINE kernel set."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_26580_b200 as P

for name, nb, reps in (("c3", 700, 40), ("c2", 2500, 100), ("c4", 300, 25)):
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, nb)
    sched = P.RevealSchedule(steps=cfg.steps)
    rm = cfg.remask or P.RemaskConfig(rank_fraction=0.25)
    ref = ctx.refine(S, wl.k, sched, rm)
    t0 = time.time()
    bad = 0
    for i in range(reps):
        g = ctx.refine(S, wl.k, sched, rm)
        if not np.array_equal(g, ref):
            bad += 1
            print(name, "iteration", i, "differs in", int((g != ref).sum()), "symbols", flush=True)
    print(f"{name}: {reps} repeated decodes of {nb} bins, {bad} differing, {time.time() - t0:.1f} s", flush=True)
    ctx.close()
    if bad:
        sys.exit(1)
