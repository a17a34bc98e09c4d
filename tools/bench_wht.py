"""The A14 kernel (batched GF(Q) check-node update in the WHT domain, cider_check_update_wht)
on a large batch, for an ncu capture of its achieved HBM bandwidth:

  ncu --set full -k regex:wht_check_update python tools/bench_wht.py [--checks 32768] [--m 8] [--d 6]

Algorithmic bytes per check = 2 x d x Q x 8 (v2c in, c2v out, fp64) + d x 4 (coefficients)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26580_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--checks", type=int, default=32768)
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--d", type=int, default=6)
a = ap.parse_args()
q = 1 << a.m
rng = np.random.default_rng(0)
v2c = rng.random((a.checks, a.d, q)) ** 3
v2c /= v2c.sum(-1, keepdims=True)
cf = rng.integers(1, q, size=(a.checks, a.d)).astype(np.int32)
P.check_update_wht(a.m, v2c[:64], cf[:64])  # warm-up (context, module load)
t0 = time.perf_counter()
out = P.check_update_wht(a.m, v2c, cf)
dt = time.perf_counter() - t0
print(json.dumps({"checks": a.checks, "Q": q, "d": a.d, "bytes_per_check": 2 * a.d * q * 8 + a.d * 4,
                  "host_call_s": round(dt, 4), "sum_ok": bool(np.allclose(out.sum(-1), 1.0))}))
