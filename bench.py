#!/usr/bin/env python3
"""Benchmark of the CIDER refinement decoder on B200 (bins decoded / s).

python bench.py --gpus N --steps K --warmup W [--config c5] [--bins-per-step B] [--impl ours|reference]

A step = one full decode (T refinement steps + gamma=0 pass + rank-25% remask pass) of one
batch of B bins per GPU. Workload: BASELINE config 5 (= config-3 bins: K=8, L=64, GF(256), N=6,
D=256, H=1024, 8 heads, T=16 + 4-step remask, bf16), bins sharded contiguously over ranks, each
rank generating its own seeded bins (derive_seed(0, 16+bin)); one NCCL all-gather of the decoded
grids at the end (the only collective). `value` times device-resident inputs with CUDA events;
`e2e` times the public host-pointer C-ABI call (H2D of S and D2H of the grids inside).
--impl reference times the reference's own CPU code (oracle/_ref) on the host cores instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import paper_2605_26580_b200 as P  # noqa: E402

METRIC = "bins_decoded_per_sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--bins-per-step", type=int, default=0, help="bins per GPU per step (0 = config default)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "fallback": True}


def kernel_rooflines(st, tot_ms, pk):
    """Per kernel class of one profiled step: algorithmic work (engine's Launch accounting: executed
    2MNK FLOPs, compulsory HBM bytes) over CUDA-event time, against the bound its arithmetic
    intensity implies (ridge = measured bf16 sustained / HBM)."""
    peak_t, peak_b = pk.get("bf16_tflops_sustained", 1360.2), pk.get("hbm_gbs", 6539.2)
    ridge = peak_t * 1e12 / (peak_b * 1e9)
    out = {}
    for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
        if v["ms"] <= 0 or 100 * v["ms"] / max(tot_ms, 1e-9) < 0.5:
            continue
        fl, by, sec = v["flops"], v["bytes"], v["ms"] / 1e3
        tensor = fl > 0 and (by <= 0 or fl / by >= ridge)
        if tensor:
            ach = fl / sec / 1e12
            out[k] = {"ms": round(v["ms"], 2), "share": round(v["ms"] / tot_ms, 4), "bound": "tensor",
                      "achieved": round(ach, 1), "unit": "TFLOP/s", "frac": round(ach / peak_t, 4)}
        elif by > 0:
            ach = by / sec / 1e9
            out[k] = {"ms": round(v["ms"], 2), "share": round(v["ms"] / tot_ms, 4), "bound": "hbm",
                      "achieved": round(ach, 1), "unit": "GB/s", "frac": round(ach / peak_b, 4)}
    return out


DEFAULT_BINS = {"c1": 64, "c2": 4096, "c3": 2048, "c4": 1024, "c5": 2048}


class Dist:
    """torch.distributed (gloo) for plumbing only: barrier, max-reduce, NCCL id broadcast."""

    def __init__(self, n):
        self.rank = int(os.environ.get("RANK", 0))
        self.world = int(os.environ.get("WORLD_SIZE", 1))
        self.local = int(os.environ.get("LOCAL_RANK", 0))
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not self.dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t)
        return float(t.item())

    def bcast_bytes(self, b: bytes) -> bytes:
        if not self.dist:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for i, nm in enumerate(names):
                if r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


def reference_sample(cfg, sample_s: float, threads: int):
    """The reference's own CPU code (oracle/_ref: ura::module_a / module_b / final_logits composed per layer,
    attention Psi from ref_shim) timed on `threads` host threads: one denoiser forward per thread on distinct
    bins, repeated until ~sample_s; bins/s = forwards/s / forwards-per-bin."""
    from oracle.binding import Checker, have_reference
    kind = "reference" if have_reference() else "port"
    chk = Checker("ref" if kind == "reference" else "oracle")
    wl, model = cfg.workload, cfg.model
    edges = wl.code()
    _, S = wl.bins(edges, 0, threads)
    w = P.model_weights_as_run(model, P.weights_init(model, 1))
    rng = np.random.default_rng(0)
    done = [0] * threads
    t_end = [0.0]

    def work(i):
        X = np.full((wl.k, wl.slots), -1, np.int32)
        X[:, : wl.slots // 2] = rng.integers(0, model.q, size=(wl.k, wl.slots // 2))
        while True:
            chk.denoise(model, w, edges, wl.checks, wl.slots, X, S[i].astype(np.float64))
            done[i] += 1
            if time.perf_counter() >= t_end[0]:
                return

    t0 = time.perf_counter()
    t_end[0] = t0 + sample_s
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    fwd = sum(done)
    per_bin = P.forward_count(cfg)
    return {"value": fwd / dt / per_bin, "unit": "bins/s", "cores": threads, "kind": kind,
            "sample": f"{fwd} denoiser forwards of {cfg.name} bins (1 per thread, ~{sample_s:.0f} s) on {threads} "
                      f"threads, x{per_bin} forwards/bin; fp64; {cpu_info()[0]}"}


def arm_config(cfg, B, world):
    """The `config` both arms report (the reference arm times a bounded sample of this workload)."""
    wl, model = cfg.workload, cfg.model
    return {"workload": f"{cfg.name}: K={wl.k} L={wl.slots} Q={model.q} N={model.layers} D={model.dim} H={model.hidden} "
                        f"heads={model.heads} T={cfg.steps}"
                        + (" + rank-25% remask" if cfg.remask else "") + f"; {B} bins/GPU/step",
            "bins_per_gpu_per_step": B, "global_batch": B * world,
            "parallelism": f"bin-sharded x{world} (no per-step collective)",
            "l2": "inputs+working set per step >> 126 MB L2 (no flush needed)",
            "forwards_per_bin": P.forward_count(cfg), "gflop_per_bin": round(P.flops_per_bin(cfg) / 1e9, 2),
            "survey_gflop_per_bin": round(P.survey_flops_per_bin(cfg) / 1e9, 2)}


def run_reference_arm(a, cfg, dist):
    if dist.rank != 0:
        return
    _, ncpu = cpu_info()
    vals = []
    for i in range(a.warmup + a.steps):
        r = reference_sample(cfg, max(3.0, a.cpu_sample_s / 2), ncpu)
        if i >= a.warmup:
            vals.append(r["value"])
    v = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "bins/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE evidence model)",
            "config": dict(arm_config(cfg, a.bins_per_step or DEFAULT_BINS[a.config], a.gpus),
                           reference_sample="each step times one fp64 denoiser forward of this workload's bins per host "
                                            "thread and scales by the forwards per bin"),
            "cpu_baseline": {"value": v, "unit": "bins/s", "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]},
            "e2e": {"value": v, "unit": "bins/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    cfg = P.configs()[a.config]
    dist = Dist(a.gpus)
    if a.impl == "reference":
        run_reference_arm(a, cfg, dist)
        dist.close()
        return
    wl, model = cfg.workload, cfg.model
    B = a.bins_per_step or DEFAULT_BINS[a.config]
    world, rank = dist.world, dist.rank
    edges = wl.code()
    w = P.weights_init(model, 1)
    ctx = P.Context(model, w, edges, wl.checks, wl.slots, device=dist.local)
    L, Q, K = wl.slots, model.q, wl.k
    lib = P.lib()
    sched = P.RevealSchedule(steps=cfg.steps)
    rmd = (cfg.remask or P.RemaskConfig()).desc()
    sd = sched.desc()

    # inputs: n_batch distinct batches of this rank's shard, resident in HBM (value) and pinned host (e2e)
    n_batch = min(a.steps + a.warmup, 4)
    s_bytes, g_bytes = B * L * Q * 4, B * K * L * 4
    hostS, devS, devG, truths = [], [], [], []
    for i in range(n_batch):
        first, _ = P.shard(0, B, rank, world, step=i)
        hp = C.c_void_p()
        P._check(lib.cider_host_alloc(s_bytes, C.byref(hp)))
        arr = np.ctypeslib.as_array((C.c_float * (B * L * Q)).from_address(hp.value)).reshape(B, L, Q)
        truth, _ = wl.bins(edges, first, B, out_S=arr)
        truths.append(truth)
        hostS.append((hp, arr))
        dp, dg = C.c_void_p(), C.c_void_p()
        P._check(lib.cider_device_alloc(ctx.h, s_bytes, C.byref(dp)))
        P._check(lib.cider_device_alloc(ctx.h, g_bytes, C.byref(dg)))
        P._check(lib.cider_memcpy_h2d(ctx.h, dp, hp, s_bytes))
        devS.append(dp)
        devG.append(dg)
    hg = C.c_void_p()
    P._check(lib.cider_host_alloc(g_bytes, C.byref(hg)))
    host_grid = np.ctypeslib.as_array((C.c_int32 * (B * K * L)).from_address(hg.value)).reshape(B, K, L)
    P._check(lib.cider_synchronize(ctx.h))

    def step_device(i):
        P._check(lib.cider_refine_device(ctx.h, B, K, devS[i % n_batch], C.byref(sd), C.byref(rmd), devG[i % n_batch]))

    def step_e2e(i):
        hp, _ = hostS[i % n_batch]
        P._check(lib.cider_refine(ctx.h, B, K, hp, C.byref(sd), C.byref(rmd), hg, None, None))

    for i in range(a.warmup):
        step_device(i)
    P._check(lib.cider_synchronize(ctx.h))

    # ---- value: device-resident inputs, CUDA events on the context stream ----
    clocks = Clocks(dist.local)
    dist.barrier()
    P._check(lib.cider_synchronize(ctx.h))
    clocks.start()
    l0 = ctx.launch_count()
    P._check(lib.cider_event_record(ctx.h, 0))
    for i in range(a.steps):
        step_device(a.warmup + i)
    P._check(lib.cider_event_record(ctx.h, 1))
    P._check(lib.cider_synchronize(ctx.h))
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    ms = C.c_float()
    P._check(lib.cider_event_elapsed(ctx.h, 0, 1, C.byref(ms)))
    dist.barrier()
    t_max = dist.max(ms.value)
    value = world * B * a.steps / (t_max / 1e3)

    # ---- e2e: public host-pointer API, H2D of S + D2H of grids inside the region ----
    e2e_steps = max(1, min(a.steps, 3))
    dist.barrier()
    P._check(lib.cider_synchronize(ctx.h))
    t0 = time.perf_counter()
    P._check(lib.cider_event_record(ctx.h, 2))
    for i in range(e2e_steps):
        step_e2e(i)
    P._check(lib.cider_event_record(ctx.h, 3))
    P._check(lib.cider_synchronize(ctx.h))
    wall = time.perf_counter() - t0
    ms2 = C.c_float()
    P._check(lib.cider_event_elapsed(ctx.h, 2, 3, C.byref(ms2)))
    e2e_ms = dist.max(max(ms2.value, wall * 1e3))
    e2e = world * B * e2e_steps / (e2e_ms / 1e3)

    # SER of this rank's first batch (from the e2e pass, batch 0), summed over ranks
    P._check(lib.cider_memcpy_d2h(ctx.h, hg, devG[0], g_bytes))
    P._check(lib.cider_synchronize(ctx.h))
    ser, cer = P.ser_cer(truths[0], host_grid)
    ser = dist.sum(ser) / world
    cer = dist.sum(cer) / world

    # ---- the one collective: NCCL all-gather of the decoded grids ----
    gather = None
    if world > 1:
        idb = C.create_string_buffer(128)
        if rank == 0:
            P._check(lib.cider_nccl_unique_id(idb))
        uid = dist.bcast_bytes(idb.raw)
        P._check(lib.cider_nccl_init(ctx.h, uid, rank, world))
        rg = C.c_void_p()
        P._check(lib.cider_device_alloc(ctx.h, g_bytes * world, C.byref(rg)))
        P._check(lib.cider_event_record(ctx.h, 4))
        P._check(lib.cider_nccl_allgather(ctx.h, devG[0], rg, g_bytes))
        P._check(lib.cider_event_record(ctx.h, 5))
        P._check(lib.cider_synchronize(ctx.h))
        gms = C.c_float()
        P._check(lib.cider_event_elapsed(ctx.h, 4, 5, C.byref(gms)))
        gather = {"bytes": g_bytes * world, "ms": gms.value}

    # ---- roofline of the dominant kernel class, from CUDA events on the launching stream ----
    ctx.reset_stats()
    ctx.set_profiling(True)
    step_device(0)
    P._check(lib.cider_synchronize(ctx.h))
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    pk = peaks()
    tot_ms = sum(v["ms"] for v in st.values())
    # the dominant kernel class of the step (all its launches), timed with CUDA events on the ctx stream
    dom_name, dom = max(st.items(), key=lambda kv: kv[1]["ms"])
    dom_launch_ms = dom["ms"] / max(dom["launches"], 1)
    tensor = dom["flops"] > 0
    per_launch = (dom["flops"] if tensor else dom["bytes"]) / max(dom["launches"], 1)  # algorithmic
    if tensor:
        achieved = per_launch / (dom_launch_ms / 1e3) / 1e12
        peak_val, unit, peak_note = pk.get("bf16_tflops_sustained", 1360.2), "TFLOP/s", \
            "measured sustained bf16 (MEASURED_PEAKS.json); kernel timed inside a long step"
    else:
        achieved = per_launch / (dom_launch_ms / 1e3) / 1e9
        peak_val, unit, peak_note = pk.get("hbm_gbs", 6539.2), "GB/s", "measured HBM copy bandwidth (MEASURED_PEAKS.json)"
    traffic, traffic_src = None, None
    try:  # DRAM bytes of this kernel class from an ncu --set full capture, per unit of algorithmic work
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        k = prof["kernels"].get(dom_name)
        if k:
            traffic = round(k["dram_bytes_per_algo_unit"] * per_launch)
            traffic_src = k["source"]
    except Exception:
        pass
    gem = {k: v for k, v in st.items() if v["flops"] > 0}
    g_ms = sum(v["ms"] for v in gem.values())
    g_fl = sum(v["flops"] for v in gem.values())
    fpb = P.flops_per_bin(cfg)
    step_tflops = fpb * value / 1e12
    top = sorted(st.items(), key=lambda kv: -kv[1]["ms"])[:16]
    roof = {"bound": "tensor" if tensor else "hbm", "achieved": round(achieved, 1), "peak": peak_val, "unit": unit,
            "frac": round(achieved / peak_val, 4), "traffic": traffic,
            "kernel": f"{dom_name}: {dom['launches']} launches/step, {dom_launch_ms:.3f} ms/launch, "
                      f"{100 * dom['ms'] / max(tot_ms, 1e-9):.1f}% of step kernel time",
            "algorithmic_per_launch": per_launch, "traffic_source": traffic_src,
            "peak_note": peak_note,
            "frac_of_burst": round(achieved / pk.get("bf16_tflops", 1638.1), 4) if tensor else None,
            "all_tensor_kernels": {"tflops": round(g_fl / (g_ms / 1e3) / 1e12, 1) if g_ms else 0.0,
                                   "share_of_step": round(g_ms / max(tot_ms, 1e-9), 4)},
            "step_algorithmic_tflops": round(step_tflops, 1),
            "step_frac": round(step_tflops / pk.get("bf16_tflops_sustained", 1360.2) / world, 4),
            "top_kernels_ms": {k: round(v["ms"], 2) for k, v in top},
            "kernels": kernel_rooflines(st, tot_ms, pk)}

    line = {"metric": METRIC, "value": round(value, 2), "unit": "bins/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(t_max / a.steps, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if model.precision == P.BF16 else "f32",
            "data": "synthetic (seeded BASELINE evidence model, random-init weights seed 1)",
            "config": arm_config(cfg, B, world),
            "e2e": {"value": round(e2e, 2), "unit": "bins/s", "h2d_bytes_per_step": s_bytes * world,
                    "d2h_bytes_per_step": g_bytes * world, "steps": e2e_steps},
            "gpu_launches": int(launches),
            "roofline": roof,
            "clocks": clk,
            "ser": round(ser, 5), "cer": round(cer, 5)}
    if gather:
        line["nccl_gather"] = gather
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            line["cpu_baseline"] = reference_sample(cfg, a.cpu_sample_s, cpu_info()[1])
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    dist.close()


if __name__ == "__main__":
    main()
