"""Diagnostic GPU probe (not a pytest module): prints parity errors and rough timings.

usage: python tests/gpu_probe.py [quick|full]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_26580_b200 as P  # noqa: E402
from oracle.binding import Checker  # noqa: E402

orc = Checker("oracle")
mode = sys.argv[1] if len(sys.argv) > 1 else "quick"


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


def parity(model, wl, nb=2, steps=4, K=None, remask=None, tag=""):
    K = K or wl.k
    edges = wl.code()
    truth, S = wl.bins(edges, 0, nb)
    w = P.weights_init(model, 1)
    wr = P.model_weights_as_run(model, w)
    ctx = P.Context(model, w, edges, wl.checks, wl.slots)
    rng = np.random.default_rng(3)
    X = rng.integers(-1, model.q, size=(nb, K, wl.slots)).astype(np.int32)
    t = time.time()
    lg, inc = ctx.denoise(X, S, want_incoming=True)
    t_dn = time.time() - t
    e_lg, e_in = 0.0, 0.0
    for b in range(nb):
        lo, io = orc.denoise(model, wr, edges, wl.checks, wl.slots, X[b], S[b].astype(np.float64), True)
        e_lg = max(e_lg, rel(lg[b], lo))
        e_in = max(e_in, rel(inc[b], io))
    sched = P.RevealSchedule(steps=steps)
    t = time.time()
    grid, fl, tr = ctx.refine(S, K, sched, remask, want_final_logits=True, want_trace=True)
    t_rf = time.time() - t
    ro = orc.refine(model, wr, edges, wl.checks, wl.slots, S.astype(np.float64), K, sched, remask, want_final_logits=True)
    same = int((grid == ro["grid"]).all(axis=(1, 2)).sum())
    print(f"[{tag}] denoise logits rel {e_lg:.2e} incoming rel {e_in:.2e} ({t_dn*1e3:.1f} ms) | refine grids equal "
          f"{same}/{nb}, final logits rel {rel(fl, ro['final_logits']):.2e}, first {tr['first_reveals'][:4]} vs "
          f"{ro['first_reveals'][:4]}, remask rows {tr['remask_rows'][:2, :2].tolist()} vs {ro['remask_rows'][:2, :2].tolist()}"
          f" ser gpu {P.ser_cer(truth, grid)} oracle {P.ser_cer(truth, ro['grid'])} ({t_rf*1e3:.1f} ms)", flush=True)


def throughput(cfg, nb, tag):
    wl, model = cfg.workload, cfg.model
    edges = wl.code()
    _, S = wl.bins(edges, 0, nb)
    w = P.weights_init(model, 1)
    ctx = P.Context(model, w, edges, wl.checks, wl.slots)
    sched = P.RevealSchedule(steps=cfg.steps)
    ctx.refine(S[: max(1, nb // 8)], wl.k, sched, cfg.remask)
    t = time.time()
    grid = ctx.refine(S, wl.k, sched, cfg.remask)
    dt = time.time() - t
    F = P.flops_per_bin(cfg) * nb
    print(f"[{tag}] {nb} bins in {dt:.3f} s -> {nb/dt:.1f} bins/s, {F/dt/1e12:.1f} TFLOP/s algorithmic", flush=True)
    ctx.set_profiling(True)
    ctx.refine(S[: max(1, nb // 4)], wl.k, sched, cfg.remask)
    st = ctx.kernel_stats()
    tot = sum(v["ms"] for v in st.values())
    for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"])[:12]:
        tf = v["flops"] / max(1e-9, v["ms"]) / 1e9
        gb = v["bytes"] / max(1e-9, v["ms"]) / 1e6
        print(f"    {k:16s} {v['ms']:9.2f} ms {100*v['ms']/tot:5.1f}%  n={v['launches']:5d}  {tf:8.1f} TF/s  {gb:8.1f} GB/s")


cf = P.configs()
print("devices", P.device_count(), flush=True)
parity(cf["c1"].model, cf["c1"].workload, nb=4, steps=4, tag="c1 fp32")
parity(P.Model.ref_exact(4, 64), cf["c1"].workload, nb=4, steps=4, tag="c1-shape ref-exact fp32")
wl8 = P.Workload(m=4, slots=16, checks=8, k=8, snr_db=4, p_erase=.1, p_false=.1)
parity(P.Model.ref_exact(4, 32), wl8, nb=3, steps=6, remask=P.RemaskConfig(thresholds=(0.3, 0.2, 0.1)), tag="thr remask fp32")
parity(P.Model.ref_exact(4, 32), wl8, nb=3, steps=6, remask=P.RemaskConfig(rank_fraction=0.25), tag="rank remask fp32")
wl6 = P.Workload(m=6, slots=16, checks=8, k=2, snr_db=6.0)
parity(P.Model(m=6, dim=64, hidden=64, layers=1, heads=0, precision=P.BF16), wl6, nb=2, tag="bf16 ref-exact-shape")
parity(P.Model(m=6, dim=128, hidden=256, layers=2, heads=4, precision=P.BF16), wl6, nb=2, tag="bf16 stacked+attn")
parity(P.Model(m=6, dim=128, hidden=256, layers=2, heads=4, precision=P.FP32), wl6, nb=2, tag="fp32 stacked+attn")
throughput(cf["c1"], 64, "c1 64 bins")
throughput(cf["c2"], 1024 if mode == "quick" else 4096, "c2")
throughput(cf["c3"], 64 if mode == "quick" else 1024, "c3")
