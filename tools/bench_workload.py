"""Evidence generation throughput: host generator (all host threads) vs the device
generator, c5 shapes. python tools/bench_workload.py [--bins 8192]"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_26580_b200 as P  # noqa: E402
import ctypes as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--bins", type=int, default=8192)
a = ap.parse_args()
wl = P.configs()[a.config].workload
e = wl.code()
m = P.Model(m=wl.m, dim=64, hidden=64)
ctx = P.Context(m, P.weights_init(m, 1), e, wl.checks, wl.slots)
wl.bins(e, 0, 64)
t0 = time.perf_counter(); wl.bins(e, 0, a.bins); host = time.perf_counter() - t0
dt, ds = wl.bins_device(ctx, e, 0, 64, copy_back=False)
P._check(P.lib().cider_device_free(ctx.h, dt)); P._check(P.lib().cider_device_free(ctx.h, ds))
t0 = time.perf_counter(); dt, ds = wl.bins_device(ctx, e, 0, a.bins, copy_back=False); dev = time.perf_counter() - t0
print(json.dumps({"metric": "evidence_bins_per_s", "config": a.config, "bins": a.bins,
                  "host": {"value": round(a.bins / host, 1), "threads": os.cpu_count()},
                  "device": {"value": round(a.bins / dev, 1), "note": "one thread per bin, synchronous call"},
                  "speedup": round(host / dev, 1)}))
