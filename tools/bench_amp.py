"""Throughput of the batched AMP slot detector against the reference's own
detect_frame on the host (oracle/_ref, one thread per frame, 16 threads).

  python tools/bench_amp.py [q n_s slots k B]      -> one JSON line
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_26580_b200 as P  # noqa: E402
from oracle.binding import Reference  # noqa: E402

q, n_s, slots, k, B = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (64, 24, 12, 2, 4096)))
ref = Reference()
dicts = ref.amp_make_dicts(q, n_s, slots, 7)
p_sym = ref.symbol_power(10.0, 24, slots)
rng = np.random.default_rng(7)
sym = rng.integers(0, q, size=(256, slots, k)).astype(np.int32)
base = np.stack([ref.amp_observe(dicts, sym[b], p_sym, 1.0, 1000 + b) for b in range(256)])
y = np.ascontiguousarray(np.tile(base, (B // 256 + 1, 1, 1))[:B])
cfg = P.AmpConfig(iters=20, rho_bg=k / q, sigma_u2=p_sym)
det = P.AmpDetector(dicts)
det.detect(y[:256], cfg)
t0 = time.perf_counter()
reps = 3
for _ in range(reps):
    S = det.detect(y, cfg)
gpu = B * reps / (time.perf_counter() - t0)
threads = min(16, os.cpu_count() or 1)
n_cpu = 64
t0 = time.perf_counter()
with ThreadPoolExecutor(threads) as ex:
    list(ex.map(lambda b: ref.amp_detect_frame(dicts, y[b], 20, cfg.rho_bg, cfg.sigma_u2, -40.0), range(n_cpu)))
cpu = n_cpu / (time.perf_counter() - t0)
print(json.dumps({"metric": "frames_detected_per_sec", "q": q, "n_s": n_s, "slots": slots, "k": k, "frames": B,
                  "gpu": round(gpu, 1), "cpu_reference": round(cpu, 1), "cpu_threads": threads,
                  "note": "host buffers in and out (H2D of y, D2H of S inside the timing); reference = ura::detect_frame"}))
