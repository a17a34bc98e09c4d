"""B200-native CIDER refinement decoder — Python mirror of the reference decoder API.

The product is ``_lib/libcider.so`` (host C++ + hand-written sm_100a CUDA) behind the C ABI in
``include/cider.h``. This module binds it with ctypes (no PyTorch on the path) and mirrors the
reference's C++ interface for the hot path (/root/reference/proj/include/ura):

  reference (C++)                                   here
  ura::DenoiserParams::random_init (denoiser.cpp:41) weights_init(model, seed)
  ura::StructuredDenoiser::logits  (denoiser.hpp:109) StructuredDenoiser(...).logits(x, s, mask_ratio)
  ura::RevealSchedule / RemaskConfig (refine.hpp:13-36) RevealSchedule / RemaskConfig
  ura::run_refinement              (refine.hpp:60-62) run_refinement(den, s, sched, k)
  ura::run_with_remasking          (refine.hpp:104)   run_with_remasking(den, s, sched, remask, k)
  ura::ser_cer                     (metrics.hpp:19-28) ser_cer(truth, pred)

Errors follow the reference: std::domain_error -> ValueError (status 3), std::runtime_error ->
RuntimeError (status 4), with the same message prefixes. There is no CPU fallback: without the
built library, or without a B200, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CIDER_LIB_DIR: load an A/B build of the library (csrc/Makefile OUT=...) instead of _lib
LIB_PATH = os.path.join(os.environ.get("CIDER_LIB_DIR") or os.path.join(_HERE, "_lib"), "libcider.so")

FP32, BF16 = 0, 1
REMASK_NONE, REMASK_THRESHOLD, REMASK_RANK = 0, 1, 2
MAX_THRESHOLDS = 8


class ModelDesc(C.Structure):
    _fields_ = [("m", C.c_int), ("prim_poly", C.c_uint32), ("dim", C.c_int), ("hidden", C.c_int),
                ("layers", C.c_int), ("heads", C.c_int), ("tau_demix", C.c_double),
                ("evidence_scale", C.c_double), ("precision", C.c_int)]


class BpConfigDesc(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("message_floor", C.c_double), ("early_exit", C.c_int)]


class AmpConfigDesc(C.Structure):
    _fields_ = [("iters", C.c_int), ("rho_bg", C.c_double), ("sigma_u2", C.c_double), ("evidence_floor", C.c_double)]


class CodeDesc(C.Structure):
    _fields_ = [("checks", C.c_int), ("slots", C.c_int), ("n_edges", C.c_int), ("edges", C.POINTER(C.c_int32))]


class ScheduleDesc(C.Structure):
    _fields_ = [("steps", C.c_int), ("tau_max", C.c_double), ("tau_min", C.c_double), ("first_reveal", C.c_int)]


class RemaskDesc(C.Structure):
    _fields_ = [("mode", C.c_int), ("n_thresholds", C.c_int), ("thresholds", C.c_double * MAX_THRESHOLDS),
                ("rank_fraction", C.c_double)]


class TraceDesc(C.Structure):
    _fields_ = [("first_reveals", C.POINTER(C.c_int32)), ("remask_rows", C.POINTER(C.c_int32)),
                ("remask_steps", C.POINTER(C.c_int32)), ("remask_mask", C.POINTER(C.c_int32)),
                ("pass_first_reveals", C.POINTER(C.c_int32)), ("n_passes", C.POINTER(C.c_int32)),
                ("max_steps", C.c_int), ("reveal_counts", C.POINTER(C.c_int32)),
                ("n_reveal_counts", C.POINTER(C.c_int32)), ("first_step_sites", C.POINTER(C.c_uint8))]


class RunConfigDesc(C.Structure):
    """cider_run_config = ura::RunConfig (dataset.hpp:19-41)."""
    _fields_ = [("scale", C.c_char * 32), ("q", C.c_int), ("l", C.c_int), ("p", C.c_int), ("col_weight", C.c_int),
                ("k", C.c_int), ("n_s", C.c_int), ("eb_db", C.c_double), ("noise_var", C.c_double), ("amp_iters", C.c_int),
                ("rho_bg", C.c_double), ("sigma_u2", C.c_double), ("evidence_floor", C.c_double), ("seed", C.c_uint64),
                ("frames", C.c_int)]


class WorkloadDesc(C.Structure):
    _fields_ = [("m", C.c_int), ("slots", C.c_int), ("checks", C.c_int), ("col_weight", C.c_int), ("k", C.c_int),
                ("snr_db", C.c_double), ("p_erase", C.c_double), ("p_false", C.c_double),
                ("master_seed", C.c_uint64)]


_lib_handle = None


def lib() -> C.CDLL:
    """Load libcider.so; raises if it was not built (there is no fallback)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libcider.so not built ({LIB_PATH}); run __graft_entry__.build()")
        h = C.CDLL(LIB_PATH)
        P = C.c_void_p
        h.cider_last_error.restype = C.c_char_p
        h.cider_weights_count.restype = C.c_size_t
        h.cider_weights_count.argtypes = [C.POINTER(ModelDesc)]
        h.cider_weights_init.argtypes = [C.POINTER(ModelDesc), C.c_uint64, P]
        h.cider_weights_init_f64.argtypes = [C.POINTER(ModelDesc), C.c_uint64, P]
        h.cider_create.argtypes = [C.POINTER(ModelDesc), P, C.POINTER(CodeDesc), C.c_int, C.POINTER(C.c_void_p)]
        h.cider_destroy.argtypes = [P]
        h.cider_destroy.restype = None
        h.cider_set_chunk.argtypes = [P, C.c_int]
        h.cider_denoise.argtypes = [P, C.c_int, C.c_int, P, P, P, P]
        h.cider_refine.argtypes = [P, C.c_int, C.c_int, P, C.POINTER(ScheduleDesc), C.POINTER(RemaskDesc), P, P,
                                   C.POINTER(TraceDesc)]
        h.cider_refine_probe.argtypes = [P, C.c_int, C.c_int, P, C.POINTER(ScheduleDesc), C.POINTER(RemaskDesc), P,
                                         C.c_int, P, C.c_int, P, P, P, C.POINTER(C.c_int)]
        h.cider_remask_pass.argtypes = [P, C.c_int, C.c_int, P, C.POINTER(ScheduleDesc), P, P, C.c_double, P, P,
                                        C.POINTER(TraceDesc)]
        h.cider_refine_ragged.argtypes = [P, C.c_int, P, P, C.c_int, P, P, P]
        h.cider_refine_device.argtypes = [P, C.c_int, C.c_int, P, C.POINTER(ScheduleDesc), C.POINTER(RemaskDesc), P]
        h.cider_device_count.argtypes = [C.POINTER(C.c_int)]
        h.cider_device_alloc.argtypes = [P, C.c_size_t, C.POINTER(C.c_void_p)]
        h.cider_device_free.argtypes = [P, P]
        h.cider_host_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p)]
        h.cider_host_free.argtypes = [P]
        h.cider_memcpy_h2d.argtypes = [P, P, P, C.c_size_t]
        h.cider_memcpy_d2h.argtypes = [P, P, P, C.c_size_t]
        h.cider_synchronize.argtypes = [P]
        h.cider_flush_l2.argtypes = [P]
        h.cider_event_record.argtypes = [P, C.c_int]
        h.cider_event_elapsed.argtypes = [P, C.c_int, C.c_int, C.POINTER(C.c_float)]
        h.cider_set_profiling.argtypes = [P, C.c_int]
        h.cider_launch_count.argtypes = [P]
        h.cider_launch_count.restype = C.c_int64
        h.cider_kernel_stats.argtypes = [P, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
        h.cider_reset_stats.argtypes = [P]
        h.cider_set_debug_guard.argtypes = [P, C.c_size_t]
        h.cider_debug_check.argtypes = [P, C.POINTER(C.c_int64)]
        h.cider_debug_poke.argtypes = [P, C.c_char_p, C.c_int64]
        h.cider_grid_pack_u8.argtypes = [P, P, P, C.c_size_t]
        h.cider_nccl_unique_id.argtypes = [C.c_char_p]
        h.cider_nccl_init.argtypes = [P, C.c_char_p, C.c_int, C.c_int]
        h.cider_nccl_allgather.argtypes = [P, P, P, C.c_size_t]
        h.cider_config_to_json.argtypes = [C.POINTER(RunConfigDesc), C.c_char_p, C.c_int]
        h.cider_config_fingerprint.argtypes = [C.POINTER(RunConfigDesc), C.c_char_p]
        h.cider_file_fingerprint.argtypes = [C.c_char_p, C.c_char_p]
        h.cider_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
        h.cider_dataset_load.argtypes = [C.c_char_p, C.POINTER(RunConfigDesc), C.c_char_p, C.c_char_p, C.POINTER(C.c_int),
                                         C.c_int, P, P, P, P]
        h.cider_workload_code.argtypes = [C.POINTER(WorkloadDesc), P]
        h.cider_workload_bins.argtypes = [C.POINTER(WorkloadDesc), P, C.c_int64, C.c_int, P, P, C.c_int]
        h.cider_save_parity_file.argtypes = [C.c_char_p, C.POINTER(CodeDesc), C.c_int, C.c_int, C.c_uint32, C.c_uint64]
        h.cider_load_parity_file.argtypes = [C.c_char_p, C.c_int, P, P, P, P, P, P, P, P]
        h.cider_workload_bins_device.argtypes = [C.POINTER(WorkloadDesc), P, C.c_int64, C.c_int, P, P, C.c_int]
        h.cider_ser_cer.argtypes = [C.c_int, C.c_int, C.c_int, P, P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        h.cider_check_update_wht.argtypes = [C.c_int, C.c_int, C.c_int, P, P, P, C.c_int]
        h.cider_bp_create.argtypes = [C.c_int, C.c_uint32, C.POINTER(CodeDesc), C.c_int, C.POINTER(C.c_void_p)]
        h.cider_bp_destroy.argtypes = [P]
        h.cider_bp_decode.argtypes = [P, C.c_int, P, C.POINTER(BpConfigDesc), P, P, P, P]
        h.cider_sic_decode.argtypes = [P, C.c_int, C.c_int, P, C.POINTER(BpConfigDesc), C.c_double, P, P, P]
        h.cider_amp_create.argtypes = [C.c_int, C.c_int, C.c_int, P, C.c_int, C.POINTER(C.c_void_p)]
        h.cider_amp_destroy.argtypes = [P]
        h.cider_amp_detect.argtypes = [P, C.c_int, P, C.POINTER(AmpConfigDesc), P]
        _lib_handle = h
    return _lib_handle


def exported_symbols() -> list:
    """Names declared in include/cider.h (used by the ABI test)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "cider.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"\b(cider_[a-z0-9_]+)\s*\(", src)))


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().cider_last_error().decode()
    if rc == 3:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- configuration ---------------------------------------------------------------------------
@dataclass
class Model:
    """Hyper-parameters (cider_model_desc). ref-exact = layers 1, hidden = dim, heads 0."""
    m: int
    dim: int
    hidden: int
    layers: int = 1
    heads: int = 0
    tau_demix: float = 1.0
    evidence_scale: float = 1.0
    precision: int = FP32
    prim_poly: int = 0

    @property
    def q(self) -> int:
        return 1 << self.m

    def desc(self) -> ModelDesc:
        return ModelDesc(self.m, self.prim_poly, self.dim, self.hidden, self.layers, self.heads, self.tau_demix,
                         self.evidence_scale, self.precision)

    @staticmethod
    def ref_exact(m: int, dim: int, precision: int = FP32) -> "Model":
        return Model(m=m, dim=dim, hidden=dim, layers=1, heads=0, precision=precision)


@dataclass
class RevealSchedule:
    """ura::RevealSchedule (refine.hpp:13-18)."""
    steps: int = 12
    tau_max: float = 1.0
    tau_min: float = 1.0
    first_reveal: bool = True

    def desc(self) -> ScheduleDesc:
        return ScheduleDesc(self.steps, self.tau_max, self.tau_min, 1 if self.first_reveal else 0)


@dataclass
class RemaskConfig:
    """ura::RemaskConfig (refine.hpp:33-36) + the rank-fraction mode of BASELINE config 3."""
    thresholds: Sequence[float] = ()
    rank_fraction: Optional[float] = None

    def desc(self) -> RemaskDesc:
        d = RemaskDesc()
        if self.rank_fraction is not None:
            d.mode = REMASK_RANK
            d.rank_fraction = float(self.rank_fraction)
        elif len(self.thresholds):
            if len(self.thresholds) > MAX_THRESHOLDS:
                raise ValueError("remask: too many thresholds")
            d.mode = REMASK_THRESHOLD
            d.n_thresholds = len(self.thresholds)
            for i, t in enumerate(self.thresholds):
                d.thresholds[i] = float(t)
        else:
            d.mode = REMASK_NONE
        return d


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round to bf16 (nearest-even) and return as float64: what BF16 mode uploads."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def model_weights_as_run(model: Model, weights: np.ndarray) -> np.ndarray:
    """The fp64 values the device actually computes with: fp32-rounded (FP32) or bf16-rounded (BF16)."""
    w = np.asarray(weights, dtype=np.float32).astype(np.float64)
    return round_bf16(w) if model.precision == BF16 else w


def weights_count(model: Model) -> int:
    d = model.desc()
    return int(lib().cider_weights_count(C.byref(d)))


def weights_init(model: Model, seed: int = 1, f64: bool = False) -> np.ndarray:
    """DenoiserParams::random_init generalised to stacked layers (flat layout of cider.h)."""
    d = model.desc()
    n = weights_count(model)
    if n == 0:
        raise ValueError("bad model dimensions")
    out = np.empty(n, dtype=np.float64 if f64 else np.float32)
    fn = lib().cider_weights_init_f64 if f64 else lib().cider_weights_init
    _check(fn(C.byref(d), C.c_uint64(seed), _ptr(out)))
    return out


def code_desc(edges: np.ndarray, checks: int, slots: int):
    e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 3)
    return CodeDesc(checks, slots, int(e.shape[0]), e.ctypes.data_as(C.POINTER(C.c_int32))), e


# ---- the context ------------------------------------------------------------------------------
class Context:
    """One cider_ctx: weights + Tanner tables resident on one B200."""

    def __init__(self, model: Model, weights: np.ndarray, edges: np.ndarray, checks: int, slots: int,
                 device: int = 0):
        self.model = model
        self.checks, self.slots = checks, slots
        self._w = np.ascontiguousarray(weights, dtype=np.float32)
        cd, self._edges = code_desc(edges, checks, slots)
        md = model.desc()
        h = C.c_void_p()
        self.device = device
        _check(lib().cider_create(C.byref(md), _ptr(self._w), C.byref(cd), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().cider_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_chunk(self, n: int):
        _check(lib().cider_set_chunk(self.h, n))

    def denoise(self, X: np.ndarray, S: np.ndarray, want_incoming: bool = False):
        """One forward for B bins. X: B x K x L int32 (-1 = MASK), S: B x L x Q."""
        X = np.ascontiguousarray(X, dtype=np.int32)
        S = np.ascontiguousarray(S, dtype=np.float32)
        B, K, L = X.shape
        q = self.model.q
        logits = np.empty((B, K, L, q), dtype=np.float32)
        inc = np.empty((B, self.model.layers, K, L, self.model.dim), dtype=np.float32) if want_incoming else None
        _check(lib().cider_denoise(self.h, B, K, _ptr(X), _ptr(S), _ptr(logits), _ptr(inc)))
        return (logits, inc) if want_incoming else logits

    def refine(self, S: np.ndarray, K: int, sched: RevealSchedule, remask: Optional[RemaskConfig] = None,
               want_final_logits: bool = False, want_trace: bool = False):
        S = np.ascontiguousarray(S, dtype=np.float32)
        B, L, q = S.shape
        grid = np.empty((B, K, L), dtype=np.int32)
        fl = np.empty((B, K, L, q), dtype=np.float32) if want_final_logits else None
        sd = sched.desc()
        rd = (remask or RemaskConfig()).desc()
        tr = None
        trd = None
        if want_trace:
            # ura::RefineTrace (refine.hpp:48-54) per bin; reveal_counts / first_step_sites describe the
            # most recent pass, pass_first_reveals every pass run (n_passes of them)
            ms = max(sched.steps, 1)
            tr = {"first_reveals": np.zeros(B, np.int32), "remask_rows": np.zeros((B, MAX_THRESHOLDS), np.int32),
                  "remask_steps": np.zeros((B, MAX_THRESHOLDS), np.int32), "remask_mask": np.zeros((B, K), np.int32),
                  "pass_first_reveals": np.zeros((B, 1 + MAX_THRESHOLDS), np.int32), "n_passes": np.zeros(B, np.int32),
                  "reveal_counts": np.zeros((B, ms), np.int32), "n_reveal_counts": np.zeros(B, np.int32),
                  "first_step_sites": np.zeros((B, K, L), np.uint8)}
            i32 = lambda k: tr[k].ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
            trd = TraceDesc(i32("first_reveals"), i32("remask_rows"), i32("remask_steps"), i32("remask_mask"),
                            i32("pass_first_reveals"), i32("n_passes"), ms, i32("reveal_counts"), i32("n_reveal_counts"),
                            tr["first_step_sites"].ctypes.data_as(C.POINTER(C.c_uint8)))
        _check(lib().cider_refine(self.h, B, K, _ptr(S), C.byref(sd), C.byref(rd), _ptr(grid), _ptr(fl),
                                  C.byref(trd) if trd is not None else None))
        out = [grid]
        if want_final_logits:
            out.append(fl)
        if want_trace:
            out.append(tr)
        return out[0] if len(out) == 1 else tuple(out)

    def remask_pass(self, S: np.ndarray, grid: np.ndarray, confidences: np.ndarray, threshold: float,
                    sched: RevealSchedule, want_final_logits: bool = False):
        """ura::remask_pass (refine.hpp:97-100) with caller row confidences (any ConfidenceScorer):
        rows with confidence < threshold are re-decoded, the rest kept bit for bit. Returns grid (and
        the pass's final logits; NaN rows for bins that had no low row)."""
        S = np.ascontiguousarray(S, dtype=np.float32)
        g = np.ascontiguousarray(grid, dtype=np.int32)
        cf = np.ascontiguousarray(confidences, dtype=np.float64)
        B, K, L = g.shape
        out = np.empty_like(g)
        fl = np.full((B, K, L, self.model.q), np.nan, np.float32) if want_final_logits else None
        sd = sched.desc()
        _check(lib().cider_remask_pass(self.h, B, K, _ptr(S), C.byref(sd), _ptr(g), _ptr(cf), float(threshold), _ptr(out),
                                       _ptr(fl), None))
        return (out, fl) if want_final_logits else out

    def refine_probe(self, S: np.ndarray, K: int, sched: RevealSchedule, remask: Optional[RemaskConfig] = None,
                     probe_bins=(0,), want_logits: bool = True, max_records: int = 0):
        """cider_refine_probe: the decode of all B bins (one device chunk) plus, for `probe_bins`, every
        forward's input grid / output logits and every pass's output grid in execution order.
        Returns (grid B x K x L, meta R x 4 {pass, t, steps, kind}, X n_probe x R x K x L,
        logits n_probe x R x K x L x Q or None)."""
        S = np.ascontiguousarray(S, dtype=np.float32)
        B, L, q = S.shape
        pb = np.ascontiguousarray(probe_bins, dtype=np.int32)
        if not max_records:
            max_records = 2 * (sched.steps + 2) + 4
        grid = np.empty((B, K, L), dtype=np.int32)
        meta = np.zeros((max_records, 4), np.int32)
        X = np.zeros((len(pb), max_records, K, L), np.int32)
        lg = np.zeros((len(pb), max_records, K, L, q), np.float32) if want_logits else None
        n = C.c_int()
        sd, rd = sched.desc(), (remask or RemaskConfig()).desc()
        _check(lib().cider_refine_probe(self.h, B, K, _ptr(S), C.byref(sd), C.byref(rd), _ptr(grid), len(pb), _ptr(pb),
                                        max_records, _ptr(meta), _ptr(X), _ptr(lg), C.byref(n)))
        r = n.value
        return grid, meta[:r], X[:, :r], (lg[:, :r] if lg is not None else None)

    def refine_ragged(self, S: np.ndarray, loads, sched_by_load, remask_by_load=None):
        """Bins of different loads K (1..k_max) in one call (cider_refine_ragged):
        sched_by_load[K-1] / remask_by_load[K-1] as a DecoderBank's per-load configs; returns the
        bins' K x L grids in input order."""
        S = np.ascontiguousarray(S, dtype=np.float32)
        B, L, _q = S.shape
        ld = np.ascontiguousarray(loads, dtype=np.int32)
        k_max = len(sched_by_load)
        sd = (ScheduleDesc * k_max)(*[x.desc() for x in sched_by_load])
        rd = None
        if remask_by_load is not None:
            rd = (RemaskDesc * k_max)(*[(x or RemaskConfig()).desc() for x in remask_by_load])
        flat = np.empty((int(ld.sum()), L), dtype=np.int32)
        _check(lib().cider_refine_ragged(self.h, B, _ptr(ld), _ptr(S), k_max, sd, rd, _ptr(flat)))
        out, o = [], 0
        for k in ld:
            out.append(flat[o:o + k])
            o += int(k)
        return out

    # debug guard bands (out-of-bounds write check, cider_set_debug_guard / cider_debug_check)
    def set_debug_guard(self, nbytes: int):
        _check(lib().cider_set_debug_guard(self.h, nbytes))

    def debug_check(self):
        n = C.c_int64()
        _check(lib().cider_debug_check(self.h, C.byref(n)))
        return n.value, lib().cider_last_error().decode()

    # instrumentation
    def launch_count(self) -> int:
        return int(lib().cider_launch_count(self.h))

    def set_profiling(self, on: bool):
        _check(lib().cider_set_profiling(self.h, 1 if on else 0))

    def reset_stats(self):
        _check(lib().cider_reset_stats(self.h))

    def kernel_stats(self) -> dict:
        out = {}
        i = 0
        name = C.create_string_buffer(128)
        while True:
            n, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            rc = lib().cider_kernel_stats(self.h, i, name, 128, C.byref(n), C.byref(ms), C.byref(fl), C.byref(by))
            if rc != 0:
                break
            out[name.value.decode()] = {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
            i += 1
        return out


# ---- reference-shaped API ------------------------------------------------------------------------
class StructuredDenoiser:
    """ura::StructuredDenoiser (denoiser.hpp:109-130) backed by a device context."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def logits(self, x: np.ndarray, s: np.ndarray, mask_ratio: float = 0.0) -> np.ndarray:
        """x: K x L (or B x K x L), s: L x Q (or B x L x Q). mask_ratio is ignored."""
        single = x.ndim == 2
        X = x[None] if single else x
        S = s[None] if single else s
        lg = self.ctx.denoise(X, S)
        return lg[0] if single else lg


def run_refinement(den: StructuredDenoiser, s: np.ndarray, sched: RevealSchedule, k: int, **kw):
    """ura::run_refinement (refine.hpp:60-62); s: L x Q or B x L x Q."""
    single = s.ndim == 2
    out = den.ctx.refine(s[None] if single else s, k, sched, None, **kw)
    if single:
        return tuple(o[0] if isinstance(o, np.ndarray) else o for o in out) if isinstance(out, tuple) else out[0]
    return out


class MaxProbScorer:
    """ura::MaxProbScorer (refine.cpp:218-225): mean over slots of the final-pass max softmax probability."""

    def score_rows(self, grid: np.ndarray, final_logits: np.ndarray) -> np.ndarray:
        lg = np.asarray(final_logits, np.float64)
        kap = 1.0 / np.exp(lg - lg.max(-1, keepdims=True)).sum(-1)
        return kap.mean(-1)


def remask_pass(den: StructuredDenoiser, s: np.ndarray, grid: np.ndarray, confidences: np.ndarray, threshold: float,
                sched: RevealSchedule, want_final_logits: bool = False):
    """ura::remask_pass (refine.hpp:97-100) on the device; s: L x Q or B x L x Q."""
    single = s.ndim == 2
    S, g, c = (s[None], grid[None], np.asarray(confidences)[None]) if single else (s, grid, confidences)
    out = den.ctx.remask_pass(S, g, c, threshold, sched, want_final_logits)
    if single:
        return tuple(o[0] for o in out) if want_final_logits else out[0]
    return out


def run_with_remasking_scored(den: StructuredDenoiser, scorer, s: np.ndarray, sched: RevealSchedule,
                              thresholds, k: int):
    """ura::run_with_remasking (refine.cpp:277-292) with any ConfidenceScorer (an object with
    score_rows(grid, final_logits) per bin): the refinement and every remask pass on the device, the
    row scores on the host between them, exactly the reference's stage loop. s: B x L x Q."""
    prev = 1.0
    for t in thresholds:  # validate_remask_config (refine.cpp:48-57)
        if t <= 0.0 or t >= 1.0:
            raise ValueError("remask thresholds must lie in (0,1)")
        if t >= prev:
            raise ValueError("remask thresholds must be strictly descending")
        prev = t
    grid, fl = den.ctx.refine(s, k, sched, None, want_final_logits=True)
    live = np.ones(len(grid), bool)
    for t in thresholds:
        conf = np.stack([np.asarray(scorer.score_rows(grid[b], fl[b]), np.float64) for b in range(len(grid))])
        low = (conf < t).any(1) & live
        live &= low  # the reference stops a bin at its first all-clear stage
        if not low.any():
            break
        idx = np.nonzero(low)[0]
        g2, fl2 = den.ctx.remask_pass(s[idx], grid[idx], conf[idx], t, sched, want_final_logits=True)
        grid[idx], fl[idx] = g2, fl2
    return grid


def run_with_remasking(den: StructuredDenoiser, s: np.ndarray, sched: RevealSchedule, remask: RemaskConfig, k: int,
                       **kw):
    """ura::run_with_remasking (refine.hpp:104-107) with the MaxProbScorer (refine.cpp:218-225)."""
    single = s.ndim == 2
    out = den.ctx.refine(s[None] if single else s, k, sched, remask, **kw)
    if single:
        return tuple(o[0] if isinstance(o, np.ndarray) else o for o in out) if isinstance(out, tuple) else out[0]
    return out


# ---- workload + metrics (host C++) ------------------------------------------------------------
@dataclass
class Workload:
    m: int
    slots: int
    checks: int
    k: int
    snr_db: float
    p_erase: float = 0.0
    p_false: float = 0.0
    col_weight: int = 3
    master_seed: int = 0

    def desc(self) -> WorkloadDesc:
        return WorkloadDesc(self.m, self.slots, self.checks, self.col_weight, self.k, self.snr_db, self.p_erase,
                            self.p_false, self.master_seed)

    def code(self) -> np.ndarray:
        e = np.empty((self.slots * self.col_weight, 3), dtype=np.int32)
        d = self.desc()
        _check(lib().cider_workload_code(C.byref(d), _ptr(e)))
        return e

    def bins(self, edges: np.ndarray, first: int, n: int, threads: int = 0, out_S: Optional[np.ndarray] = None):
        d = self.desc()
        edges = np.ascontiguousarray(edges, dtype=np.int32)
        truth = np.empty((n, self.k, self.slots), dtype=np.int32)
        S = out_S if out_S is not None else np.empty((n, self.slots, 1 << self.m), dtype=np.float32)
        _check(lib().cider_workload_bins(C.byref(d), _ptr(edges), first, n, _ptr(truth), _ptr(S), threads))
        return truth, S

    def bins_device(self, ctx: "Context", edges: np.ndarray, first: int, n: int, copy_back: bool = True):
        """The same bins generated on the device into buffers of `ctx`; returns host
        copies (truth, S) or, with copy_back=False, the device pointers (the caller frees them)."""
        d = self.desc()
        edges = np.ascontiguousarray(edges, dtype=np.int32)
        q = 1 << self.m
        tb, sb = n * self.k * self.slots * 4, n * self.slots * q * 4
        dt, ds = C.c_void_p(), C.c_void_p()
        _check(lib().cider_device_alloc(ctx.h, tb, C.byref(dt)))
        _check(lib().cider_device_alloc(ctx.h, sb, C.byref(ds)))
        _check(lib().cider_workload_bins_device(C.byref(d), _ptr(edges), first, n, dt, ds, ctx.device))
        if not copy_back:
            return dt, ds
        truth = np.empty((n, self.k, self.slots), dtype=np.int32)
        S = np.empty((n, self.slots, q), dtype=np.float32)
        _check(lib().cider_memcpy_d2h(ctx.h, _ptr(truth), dt, tb))
        _check(lib().cider_memcpy_d2h(ctx.h, _ptr(S), ds, sb))
        _check(lib().cider_synchronize(ctx.h))
        _check(lib().cider_device_free(ctx.h, dt))
        _check(lib().cider_device_free(ctx.h, ds))
        return truth, S


def save_parity_file(path: str, edges, checks: int, slots: int, q: int, col_weight: int = 0, prim_poly: int = 0,
                     seed: int = 0) -> None:
    """ura::save_parity_file (ldpc.cpp:197-205)."""
    cd, _e = code_desc(edges, checks, slots)
    _check(lib().cider_save_parity_file(path.encode(), C.byref(cd), q, col_weight, prim_poly, seed))


def load_parity_file(path: str, max_edges: int = 1 << 16) -> dict:
    """ura::load_parity_file (ldpc.cpp:207-226): edges sorted (check, slot) + header fields."""
    e = np.empty((max_edges, 3), np.int32)
    v = [C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_uint32(), C.c_uint64()]
    _check(lib().cider_load_parity_file(path.encode(), max_edges, _ptr(e), *[C.byref(x) for x in v]))
    n = v[0].value
    return {"edges": e[:n].copy(), "checks": v[1].value, "slots": v[2].value, "q": v[3].value,
            "col_weight": v[4].value, "prim_poly": v[5].value, "seed": v[6].value}


# ---- the reference's dataset format ----------------------------------------------
RUN_CONFIG_FIELDS = ("scale", "q", "l", "p", "col_weight", "k", "n_s", "eb_db", "noise_var", "amp_iters", "rho_bg",
                     "sigma_u2", "evidence_floor", "seed", "frames")


def run_config(**kw) -> RunConfigDesc:
    """ura::RunConfig with its defaults (dataset.hpp:19-36), overridden by `kw`."""
    d = dict(scale="tiny", q=64, l=12, p=8, col_weight=3, k=2, n_s=24, eb_db=10.0, noise_var=1.0, amp_iters=20,
             rho_bg=-1.0, sigma_u2=-1.0, evidence_floor=-40.0, seed=1, frames=100)
    d.update(kw)
    d["scale"] = d["scale"].encode()
    return RunConfigDesc(*[d[f] for f in RUN_CONFIG_FIELDS])


def config_to_json(cfg: RunConfigDesc) -> str:
    buf = C.create_string_buffer(2048)
    _check(lib().cider_config_to_json(C.byref(cfg), buf, 2048))
    return buf.value.decode()


def config_fingerprint(cfg: RunConfigDesc) -> str:
    buf = C.create_string_buffer(17)
    _check(lib().cider_config_fingerprint(C.byref(cfg), buf))
    return buf.value.decode()


def format_double(x: float) -> str:
    """format_double (dataset.cpp:57-61): the shortest round-trip decimal form (std::to_chars)."""
    buf = C.create_string_buffer(64)
    _check(lib().cider_format_double(float(x), buf, 64))
    return buf.value.decode()


def load_dataset(path: str) -> dict:
    """ura::load_dataset (dataset.cpp:176-220): {config, fingerprint, h_fingerprint, seeds, truth n x K x L,
    evidence n x L x Q (fp64), snr_db}."""
    cfg = RunConfigDesc()
    fp, hfp = C.create_string_buffer(17), C.create_string_buffer(17)
    n = C.c_int()
    _check(lib().cider_dataset_load(path.encode(), C.byref(cfg), fp, hfp, C.byref(n), 0, None, None, None, None))
    k, L, q = cfg.k, cfg.l, cfg.q
    seeds = np.empty(n.value, np.uint64)
    truth = np.empty((n.value, k, L), np.int32)
    ev = np.empty((n.value, L, q), np.float64)
    snr = np.empty(n.value, np.float64)
    _check(lib().cider_dataset_load(path.encode(), C.byref(cfg), fp, hfp, C.byref(n), n.value, _ptr(seeds), _ptr(truth),
                                    _ptr(ev), _ptr(snr)))
    conf = {f: getattr(cfg, f) for f in RUN_CONFIG_FIELDS}
    conf["scale"] = conf["scale"].decode()
    return {"config": conf, "fingerprint": fp.value.decode(), "h_fingerprint": hfp.value.decode(), "seeds": seeds,
            "truth": truth, "evidence": ev, "snr_db": snr}


def ser_cer(truth: np.ndarray, pred: np.ndarray):
    """Mean permutation-invariant SER/CER over bins (ura::ser_cer, metrics.cpp:124-145)."""
    truth = np.ascontiguousarray(truth, dtype=np.int32)
    pred = np.ascontiguousarray(pred, dtype=np.int32)
    if truth.ndim == 2:
        truth, pred = truth[None], pred[None]
    n, K, L = truth.shape
    s, c = C.c_double(), C.c_double()
    _check(lib().cider_ser_cer(n, K, L, _ptr(truth), _ptr(pred), C.byref(s), C.byref(c)))
    return s.value / n, c.value / n


def check_update_wht(m: int, v2c: np.ndarray, coeffs: np.ndarray, device: int = 0) -> np.ndarray:
    """All extrinsic check-to-variable messages of a batch of GF(2^m) checks, WHT domain
    (= ura::update_check_wht, bp.cpp:222-269). v2c: n x d x Q fp64, coeffs: n x d."""
    v = np.ascontiguousarray(v2c, dtype=np.float64)
    cf = np.ascontiguousarray(coeffs, dtype=np.int32)
    n, d, q = v.shape
    out = np.empty_like(v)
    _check(lib().cider_check_update_wht(m, n, d, _ptr(v), _ptr(cf), _ptr(out), device))
    return out


@dataclass
class BpConfig:
    """ura::BpConfig (bp.hpp:20-25); the device decoder implements the WHT backend."""
    max_iters: int = 50
    message_floor: float = 1e-30
    early_exit: bool = True

    def desc(self) -> BpConfigDesc:
        return BpConfigDesc(self.max_iters, self.message_floor, int(self.early_exit))


class BpDecoder:
    """Batched GF(Q) FFT-BP on the device: the reference's bp_decode / sic_decode
    (bp.cpp:271-368) for many bins at once, WHT-domain check updates (double-double spectra)."""

    def __init__(self, m: int, edges: np.ndarray, checks: int, slots: int, device: int = 0, prim_poly: int = 0):
        self.m, self.q, self.slots = m, 1 << m, slots
        cd, self._keep = code_desc(edges, checks, slots)
        h = C.c_void_p()
        _check(lib().cider_bp_create(m, prim_poly, C.byref(cd), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().cider_bp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bp_decode(self, lam: np.ndarray, cfg: BpConfig = BpConfig()):
        """lam: B x L x Q slot beliefs -> (hard B x L, marginals B x L x Q, converged B, iters B)."""
        lam = np.ascontiguousarray(lam, np.float64)
        B = lam.shape[0]
        hard = np.empty((B, self.slots), np.int32)
        marg = np.empty((B, self.slots, self.q), np.float64)
        conv = np.empty(B, np.int32)
        its = np.empty(B, np.int32)
        d = cfg.desc()
        _check(lib().cider_bp_decode(self.h, B, _ptr(lam), C.byref(d), _ptr(hard), _ptr(marg), _ptr(conv), _ptr(its)))
        return hard, marg, conv.astype(bool), its

    def sic_decode(self, S: np.ndarray, k: int, cfg: BpConfig = BpConfig(), cancel_value: float = float("nan")):
        """S: B x L x Q evidence -> (grid B x k x L in decode order, stage converged B x k, stage iters B x k)."""
        S = np.ascontiguousarray(S, np.float64)
        B = S.shape[0]
        grid = np.empty((B, k, self.slots), np.int32)
        sc = np.empty((B, k), np.int32)
        si = np.empty((B, k), np.int32)
        d = cfg.desc()
        _check(lib().cider_sic_decode(self.h, B, k, _ptr(S), C.byref(d), cancel_value, _ptr(grid), _ptr(sc), _ptr(si)))
        return grid, sc.astype(bool), si


@dataclass
class AmpConfig:
    """ura::AmpConfig (amp.hpp:14-19); default_amp_config sets rho_bg = K/Q, sigma_u2 = P_sym (amp.cpp:29-36)."""
    iters: int = 20
    rho_bg: float = 0.03125
    sigma_u2: float = 20.0
    evidence_floor: float = -40.0

    def desc(self) -> AmpConfigDesc:
        return AmpConfigDesc(self.iters, self.rho_bg, self.sigma_u2, self.evidence_floor)


class AmpDetector:
    """Batched AMP slot detector on the device: the reference's detect_frame
    (amp.cpp:133-148) for many frames at once. dicts: L x q x n_s complex (the per-slot
    ura::SensingMatrix columns, fixed per dataset)."""

    def __init__(self, dicts: np.ndarray, device: int = 0):
        dicts = np.ascontiguousarray(dicts, np.complex128)
        self.L, self.q, self.n_s = dicts.shape
        h = C.c_void_p()
        _check(lib().cider_amp_create(self.L, self.q, self.n_s, _ptr(dicts), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().cider_amp_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def detect(self, y: np.ndarray, cfg: AmpConfig = AmpConfig()) -> np.ndarray:
        """y: B x L x n_s complex observations -> S: B x L x q evidence rows (fp64)."""
        y = np.ascontiguousarray(y, np.complex128)
        B = y.shape[0]
        S = np.empty((B, self.L, self.q), np.float64)
        d = cfg.desc()
        _check(lib().cider_amp_detect(self.h, B, _ptr(y), C.byref(d), _ptr(S)))
        return S


def device_count() -> int:
    n = C.c_int()
    _check(lib().cider_device_count(C.byref(n)))
    return n.value


# ---- BASELINE.json configurations ----------------------------------------------------------------
@dataclass
class Config:
    name: str
    workload: Workload
    model: Model
    bins: int
    steps: int
    remask: Optional[RemaskConfig] = None
    extra: dict = field(default_factory=dict)


def configs() -> dict:
    """The five BASELINE.json configs (SURVEY §8 shape key)."""
    c1 = Config("c1", Workload(m=4, slots=16, checks=8, k=2, snr_db=10.0),
                Model(m=4, dim=64, hidden=256, layers=2, heads=4, precision=FP32), bins=64, steps=4)
    c2 = Config("c2", Workload(m=6, slots=32, checks=16, k=4, snr_db=6.0, p_erase=0.05, p_false=0.05),
                Model(m=6, dim=128, hidden=512, layers=4, heads=8, precision=BF16), bins=4096, steps=8)
    c3 = Config("c3", Workload(m=8, slots=64, checks=32, k=8, snr_db=4.0, p_erase=0.1, p_false=0.1),
                Model(m=8, dim=256, hidden=1024, layers=6, heads=8, precision=BF16), bins=16384, steps=16,
                remask=RemaskConfig(rank_fraction=0.25))
    c4 = Config("c4", Workload(m=6, slots=256, checks=128, k=4, snr_db=6.0, p_erase=0.05, p_false=0.05),
                Model(m=6, dim=256, hidden=1024, layers=6, heads=8, precision=BF16), bins=8192, steps=16)
    c5 = Config("c5", c3.workload, c3.model, bins=262144, steps=16, remask=RemaskConfig(rank_fraction=0.25))
    return {c.name: c for c in (c1, c2, c3, c4, c5)}


def forward_count(cfg: Config) -> int:
    """Denoiser forwards per bin: T + 1, plus T_rm + 1 when remasking (refine.cpp:23-26, 180-185)."""
    f = cfg.steps + 1
    if cfg.remask is not None and cfg.remask.rank_fraction:
        k_low = int(np.floor(cfg.remask.rank_fraction * cfg.workload.k))
        if k_low > 0:
            f += max(1, (cfg.steps * k_low) // cfg.workload.k) + 1
    return f


def flops_per_bin(cfg: Config) -> float:
    """Executed tensor-core FLOPs per decoded bin:
    F = 2 fwd [N (4KLQD + 6KLDH + 2K|E|QD + 2K|E|DH) + KLQD]  (SURVEY §8(d) without its attention
    D^2 key-projection term: the device computes attention scores through u_h = Wk_h^T q_h)."""
    w, m = cfg.workload, cfg.model
    K, L, Q, D, H, N = w.k, w.slots, m.q, m.dim, m.hidden, m.layers
    E = L * w.col_weight
    per = N * (4 * K * L * Q * D + 6 * K * L * D * H + 2 * K * E * Q * D + 2 * K * E * D * H) + K * L * Q * D
    return 2.0 * forward_count(cfg) * per


def survey_flops_per_bin(cfg: Config) -> float:
    """SURVEY §8(d)'s formula including F_attn = N K|E| (2D^2 + 2(d_c-1)D) (informational)."""
    w, m = cfg.workload, cfg.model
    K, E, D, N = w.k, w.slots * w.col_weight, m.dim, m.layers
    dc = E / w.checks
    extra = N * K * E * (2 * D * D + 2 * (dc - 1) * D) if m.heads else 0.0
    return flops_per_bin(cfg) + 2.0 * forward_count(cfg) * extra


def shard(first_bin: int, n_bins: int, rank: int, world: int, step: int = 0):
    """Contiguous bin shard of `rank` for `step`: [start, start + n_bins)."""
    return first_bin + (step * world + rank) * n_bins, n_bins
