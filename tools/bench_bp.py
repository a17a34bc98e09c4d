"""Benchmark of the batched GF(Q) FFT-BP decoder: SIC-BP bins/s on the device vs the
reference's own sic_decode (oracle/_ref, fp64 + long double spectra) on the host cores, same bins.

  python tools/bench_bp.py [--config c3] [--bins 512] [--iters 50] [--cpu-bins 16]

Prints one JSON line. The GPU number is end to end through cider_sic_decode (host evidence in, host
grids out); the CPU number uses one reference decode per host thread (ctypes releases the GIL).
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_26580_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bins", type=int, default=512)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--cpu-bins", type=int, default=16)
    ap.add_argument("--profile", action="store_true", help="one 2-iteration decode of --bins bins only (for ncu)")
    a = ap.parse_args()
    cfg = P.configs()[a.config]
    wl = cfg.workload
    e = wl.code()
    nb = a.bins
    truth, S = wl.bins(e, 0, nb)
    S = S.astype(np.float64)
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    bc = P.BpConfig(max_iters=a.iters)
    if not a.profile:
        dec.sic_decode(S[: min(nb, 8)], wl.k, bc)  # warm-up
    if a.profile:  # one 2-iteration decode of the whole batch: realistic launch sizes for ncu
        dec.sic_decode(S, wl.k, P.BpConfig(max_iters=2))
        return
    t0 = time.perf_counter()
    grid, sc, si = dec.sic_decode(S, wl.k, bc)
    gpu_s = time.perf_counter() - t0
    ser = float(np.mean([P.ser_cer(truth[b:b + 1], grid[b:b + 1])[0] for b in range(min(nb, 64))]))
    line = {"metric": "sic_bp_bins_per_s", "config": a.config, "bins": nb, "max_iters": a.iters,
            "shape": {"Q": 1 << wl.m, "L": wl.slots, "P": wl.checks, "K": wl.k},
            "gpu": {"value": round(nb / gpu_s, 2), "seconds": round(gpu_s, 3),
                    "mean_stage_iters": round(float(si.mean()), 2), "converged_stage_frac": round(float(sc.mean()), 4),
                    "ser_first_64": round(ser, 4)}}
    try:
        from oracle.binding import Reference, have_reference
        if have_reference() and a.cpu_bins > 0:
            ref = Reference()
            cores = os.cpu_count() or 1
            n = min(a.cpu_bins, nb)
            out = [None] * n

            def work(i0):
                for b in range(i0, n, cores):
                    out[b] = ref.sic_decode(wl.m, e, wl.checks, wl.slots, S[b:b + 1], wl.k, max_iters=a.iters)
            t0 = time.perf_counter()
            th = [threading.Thread(target=work, args=(i,)) for i in range(min(cores, n))]
            for t in th:
                t.start()
            for t in th:
                t.join()
            cpu_s = time.perf_counter() - t0
            same = sum(int(np.array_equal(out[b][0][0], grid[b])) for b in range(n))
            line["cpu_reference"] = {"value": round(n / cpu_s, 3), "bins": n, "seconds": round(cpu_s, 2),
                                     "cores": min(cores, n), "kind": "reference (oracle/_ref, bp.cpp)",
                                     "grids_identical": f"{same}/{n}"}
            line["speedup"] = round(line["gpu"]["value"] / line["cpu_reference"]["value"], 1)
    except Exception as ex:  # reported, never fatal
        line["cpu_reference"] = {"error": str(ex)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
