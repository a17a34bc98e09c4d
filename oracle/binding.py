"""ctypes bindings of the CHECKERS — test infrastructure only.

  restatement : oracle/_build/libcider_oracle.so  (cider_oracle.cpp, this repo's fp64 CPU oracle)
  reference   : oracle/_ref/libura_ref.so         (the reference's own sources + ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module; the product path (paper_2605_26580_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from paper_2605_26580_b200 import (MAX_THRESHOLDS, Model, ModelDesc, CodeDesc, RemaskConfig, RemaskDesc,
                                   RevealSchedule, ScheduleDesc, code_desc)

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(_HERE, "_build", "libcider_oracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libura_ref.so")

_handles = {}


def _load(path: str, prefix: str) -> C.CDLL:
    if path in _handles:
        return _handles[path]
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    h = C.CDLL(path)
    P = C.c_void_p
    getattr(h, f"{prefix}_last_error").restype = C.c_char_p
    d = getattr(h, f"{prefix}_denoise")
    d.argtypes = [C.POINTER(ModelDesc), P, C.POINTER(CodeDesc), C.c_int, P, P, P, P]
    if prefix == "oracle":
        h.oracle_denoise_batch.argtypes = [C.POINTER(ModelDesc), P, C.POINTER(CodeDesc), C.c_int, C.c_int, P, P, P,
                                           C.c_int]
    r = getattr(h, f"{prefix}_refine")
    r.argtypes = [C.POINTER(ModelDesc), P, C.POINTER(CodeDesc), C.c_int, C.c_int, P, C.POINTER(ScheduleDesc),
                  C.POINTER(RemaskDesc), P, P, P, P, P, P, C.c_int]
    rp = getattr(h, f"{prefix}_remask_pass")
    rp.argtypes = [C.POINTER(ModelDesc), P, C.POINTER(CodeDesc), C.c_int, C.c_int, P, C.POINTER(ScheduleDesc), P, P,
                   C.c_double, P, P, C.c_int]
    rv = getattr(h, f"{prefix}_reveal_step")
    rv.argtypes = [C.c_int, C.c_int, C.c_int, P, P, C.c_int, C.c_double, C.c_int, P]
    w = getattr(h, f"{prefix}_check_update_wht")
    w.argtypes = [C.c_int, C.c_int, P, P, C.c_int, P]
    if prefix == "ref":
        h.ref_random_init.argtypes = [C.c_int, C.c_int, C.c_uint64, P]
        h.ref_build_ldpc.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, P]
        h.ref_sample_codewords.argtypes = [C.c_int, C.POINTER(CodeDesc), C.c_int, C.c_uint64, P]
        h.ref_ser_cer.argtypes = [C.c_int, C.c_int, P, P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        h.ref_check_update_direct.argtypes = [C.c_int, C.c_int, P, P, C.c_int, P]
        h.ref_cosine_target.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        h.ref_infer_temperature.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        h.ref_infer_temperature.restype = C.c_double
        h.ref_remask_steps.argtypes = [C.c_int, C.c_int, C.c_int]
        h.ref_save_parity_file.argtypes = [C.c_char_p, C.c_int, C.POINTER(CodeDesc), C.c_int, C.c_uint32, C.c_uint64]
        h.ref_load_parity_file.argtypes = [C.c_char_p, C.c_int, P, P, P, P, P, P, P, P]
        h.ref_bp_decode.argtypes = [C.c_int, C.POINTER(CodeDesc), C.c_int, P, C.c_int, C.c_double, C.c_int, P, P, P, P]
        h.ref_weights_init.argtypes = [C.POINTER(ModelDesc), C.c_uint64, P]
        h.ref_workload_bins.argtypes = [C.c_int, C.POINTER(CodeDesc), C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_uint64, C.c_int64, C.c_int, P, P, C.c_int]
        h.ref_session_create.argtypes = [C.POINTER(ModelDesc), P, C.POINTER(CodeDesc), C.c_int, C.c_int, P,
                                         C.POINTER(ScheduleDesc), C.POINTER(RemaskDesc), C.c_int, C.POINTER(C.c_void_p)]
        h.ref_session_advance.argtypes = [P, C.c_int]
        h.ref_session_status.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), P, P]
        h.ref_session_destroy.argtypes = [P]
        h.ref_session_destroy.restype = None
        h.ref_sic_decode.argtypes = [C.c_int, C.POINTER(CodeDesc), C.c_int, C.c_int, P, C.c_int, C.c_double, C.c_int,
                                     C.c_double, P, P, P]
    _handles[path] = h
    return h


def have_reference() -> bool:
    return os.path.exists(REF_PATH)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Checker:
    """The same C-ABI served by the restatement ('oracle') or the reference itself ('ref')."""

    def __init__(self, kind: str = "oracle"):
        self.kind = kind
        self.prefix = "oracle" if kind == "oracle" else "ref"
        self.h = _load(ORACLE_PATH if kind == "oracle" else REF_PATH, self.prefix)

    def _check(self, rc: int):
        if rc == 0:
            return
        msg = getattr(self.h, f"{self.prefix}_last_error")().decode()
        if rc == 3:
            raise ValueError(msg)
        raise RuntimeError(msg)

    def denoise(self, model: Model, weights: np.ndarray, edges: np.ndarray, checks: int, slots: int,
                X: np.ndarray, S: np.ndarray, want_incoming: bool = False):
        """One bin: X K x L, S L x Q (fp64) -> logits K x L x Q (+ incoming layers x K x L x D)."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        cd, _e = code_desc(edges, checks, slots)
        X = np.ascontiguousarray(X, dtype=np.int32)
        S = np.ascontiguousarray(S, dtype=np.float64)
        K, L = X.shape
        lg = np.empty((K, L, model.q), dtype=np.float64)
        inc = np.empty((model.layers, K, L, model.dim), dtype=np.float64) if want_incoming else None
        md = model.desc()
        self._check(getattr(self.h, f"{self.prefix}_denoise")(C.byref(md), _p(w), C.byref(cd), K, _p(X), _p(S),
                                                              _p(lg), _p(inc)))
        return (lg, inc) if want_incoming else lg

    def denoise_batch(self, model: Model, weights: np.ndarray, edges: np.ndarray, checks: int, slots: int,
                      X: np.ndarray, S: np.ndarray, threads: int = 0) -> np.ndarray:
        """B independent forwards on `threads` host threads (restatement only): X B x K x L, S B x L x Q
        -> logits B x K x L x Q (fp64), bit-identical to B denoise() calls."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        cd, _e = code_desc(edges, checks, slots)
        X = np.ascontiguousarray(X, dtype=np.int32)
        S = np.ascontiguousarray(S, dtype=np.float64)
        B, K, L = X.shape
        lg = np.empty((B, K, L, model.q), dtype=np.float64)
        md = model.desc()
        self._check(self.h.oracle_denoise_batch(C.byref(md), _p(w), C.byref(cd), B, K, _p(X), _p(S), _p(lg), threads))
        return lg

    def refine(self, model: Model, weights: np.ndarray, edges: np.ndarray, checks: int, slots: int, S: np.ndarray,
               K: int, sched: RevealSchedule, remask: Optional[RemaskConfig] = None, threads: int = 0,
               want_final_logits: bool = False):
        """B bins: S B x L x Q (fp64) -> dict(grid, final_logits, first_reveals, remask_rows, remask_steps, mask)."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        cd, _e = code_desc(edges, checks, slots)
        S = np.ascontiguousarray(S, dtype=np.float64)
        B, L, q = S.shape
        out = {
            "grid": np.empty((B, K, L), np.int32),
            "final_logits": np.empty((B, K, L, q), np.float64) if want_final_logits else None,
            "first_reveals": np.zeros(B, np.int32),
            "remask_rows": np.zeros((B, MAX_THRESHOLDS), np.int32),
            "remask_steps": np.zeros((B, MAX_THRESHOLDS), np.int32),
            "remask_mask": np.zeros((B, K), np.int32),
        }
        md, sd, rd = model.desc(), sched.desc(), (remask or RemaskConfig()).desc()
        self._check(getattr(self.h, f"{self.prefix}_refine")(
            C.byref(md), _p(w), C.byref(cd), B, K, _p(S), C.byref(sd), C.byref(rd), _p(out["grid"]),
            _p(out["final_logits"]), _p(out["first_reveals"]), _p(out["remask_rows"]), _p(out["remask_steps"]),
            _p(out["remask_mask"]), threads))
        return out

    def remask_pass(self, model: Model, weights: np.ndarray, edges: np.ndarray, checks: int, slots: int, S: np.ndarray,
                    grid: np.ndarray, conf: np.ndarray, threshold: float, sched: RevealSchedule, threads: int = 0):
        """remask_pass (refine.cpp:238-275) with caller confidences for B bins -> (grid, final logits or NaN)."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        cd, _e = code_desc(edges, checks, slots)
        S = np.ascontiguousarray(S, dtype=np.float64)
        g = np.ascontiguousarray(grid, dtype=np.int32)
        cf = np.ascontiguousarray(conf, dtype=np.float64)
        B, K, L = g.shape
        out = np.empty_like(g)
        fl = np.full((B, K, L, S.shape[-1]), np.nan)
        sd = sched.desc()
        self._check(getattr(self.h, f"{self.prefix}_remask_pass")(C.byref(model.desc()), _p(w), C.byref(cd), B, K, _p(S),
                                                                  C.byref(sd), _p(g), _p(cf), threshold, _p(out), _p(fl),
                                                                  threads))
        return out, fl

    def reveal_step(self, X: np.ndarray, logits: np.ndarray, target: int, tau: float, first: bool):
        X = np.ascontiguousarray(X, dtype=np.int32)
        lg = np.ascontiguousarray(logits, dtype=np.float64)
        K, L = X.shape
        out = np.empty_like(X)
        self._check(getattr(self.h, f"{self.prefix}_reveal_step")(K, L, lg.shape[-1], _p(X), _p(lg), target, tau,
                                                                  1 if first else 0, _p(out)))
        return out

    def check_update_wht(self, m: int, incoming: np.ndarray, coeffs, target: int):
        inc = np.ascontiguousarray(incoming, dtype=np.float64)
        cf = np.ascontiguousarray(coeffs, dtype=np.int32)
        out = np.empty(1 << m, np.float64)
        self._check(getattr(self.h, f"{self.prefix}_check_update_wht")(m, inc.shape[0], _p(inc), _p(cf), target,
                                                                       _p(out)))
        return out


class Reference(Checker):
    """Extra entry points only the reference shim has (weights, code construction, metrics)."""

    def __init__(self):
        super().__init__("ref")

    def random_init(self, q: int, dim: int, seed: int) -> np.ndarray:
        n = (q + 1) * dim + 2 * q * dim + 3 * dim * 2 * dim + 3 * dim + dim * dim + dim + dim * dim + dim * 2 + dim * dim
        # exact count: embed + out_proj + sym_embed + gate(2D->D->D) + agg(D->D->D) + fuse(2D->D->D)
        n = (q + 1) * dim + 2 * q * dim + (dim * 2 * dim + dim + dim * dim + dim) * 2 + (dim * dim + dim + dim * dim + dim)
        out = np.empty(n, np.float64)
        self._check(self.h.ref_random_init(q, dim, C.c_uint64(seed), _p(out)))
        return out

    def weights_init(self, model: Model, seed: int) -> np.ndarray:
        """cider.h's flat weight layout drawn with the reference's own seeding (ref_weights_init)."""
        n = (model.q + 1) * model.dim + 2 * model.q * model.dim
        D, H = model.dim, model.hidden
        n += model.layers * ((H * 2 * D + H + D * H + D) * 2 + (H * D + H + D * H + D))
        if model.heads:
            n += model.layers * (D + D * D)
        out = np.empty(n, np.float64)
        md = model.desc()
        self._check(self.h.ref_weights_init(C.byref(md), C.c_uint64(seed), _p(out)))
        return out

    def workload_bins(self, wl, edges: np.ndarray, first: int, n: int, threads: int = 0):
        """The BASELINE evidence model over the reference's own sample_codewords (ref_workload_bins):
        (truth n x K x L, S n x L x Q fp64 holding fp32-rounded values)."""
        cd, _e = code_desc(edges, wl.checks, wl.slots)
        truth = np.empty((n, wl.k, wl.slots), np.int32)
        S = np.empty((n, wl.slots, 1 << wl.m), np.float64)
        self._check(self.h.ref_workload_bins(wl.m, C.byref(cd), wl.k, wl.snr_db, wl.p_erase, wl.p_false,
                                             C.c_uint64(wl.master_seed), first, n, _p(truth), _p(S), threads))
        return truth, S

    def build_ldpc(self, m: int, slots: int, checks: int, col_weight: int, seed: int) -> np.ndarray:
        e = np.empty((slots * col_weight, 3), np.int32)
        self._check(self.h.ref_build_ldpc(m, slots, checks, col_weight, C.c_uint64(seed), _p(e)))
        return e

    def sample_codewords(self, m: int, edges: np.ndarray, checks: int, slots: int, k: int, seed: int) -> np.ndarray:
        cd, _e = code_desc(edges, checks, slots)
        out = np.empty((k, slots), np.int32)
        self._check(self.h.ref_sample_codewords(m, C.byref(cd), k, C.c_uint64(seed), _p(out)))
        return out

    def ser_cer(self, truth: np.ndarray, pred: np.ndarray):
        t = np.ascontiguousarray(truth, np.int32)
        p = np.ascontiguousarray(pred, np.int32)
        s, c = C.c_double(), C.c_double()
        self._check(self.h.ref_ser_cer(t.shape[0], t.shape[1], _p(t), _p(p), C.byref(s), C.byref(c)))
        return s.value, c.value

    def check_update_direct(self, m: int, incoming: np.ndarray, coeffs, target: int):
        inc = np.ascontiguousarray(incoming, dtype=np.float64)
        cf = np.ascontiguousarray(coeffs, dtype=np.int32)
        out = np.empty(1 << m, np.float64)
        self._check(self.h.ref_check_update_direct(m, inc.shape[0], _p(inc), _p(cf), target, _p(out)))
        return out


    def save_parity_file(self, path: str, m: int, edges, checks: int, slots: int, col_weight: int, prim_poly: int, seed: int):
        cd, _e = code_desc(edges, checks, slots)
        self._check(self.h.ref_save_parity_file(path.encode(), m, C.byref(cd), col_weight, prim_poly, seed))

    def load_parity_file(self, path: str, max_edges: int = 1 << 16):
        e = np.empty((max_edges, 3), np.int32)
        v = [C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_uint32(), C.c_uint64()]
        self._check(self.h.ref_load_parity_file(path.encode(), max_edges, _p(e), *[C.byref(x) for x in v]))
        n = v[0].value
        return {"edges": e[:n].copy(), "checks": v[1].value, "slots": v[2].value, "q": v[3].value,
                "col_weight": v[4].value, "prim_poly": v[5].value, "seed": v[6].value}

    def bp_decode(self, m: int, edges: np.ndarray, checks: int, slots: int, lam: np.ndarray, max_iters: int = 50,
                  message_floor: float = 1e-30, early_exit: bool = True):
        """ura::bp_decode (bp.cpp:271-347), WHT backend, per bin: (hard, marginals, converged, iters)."""
        cd, _e = code_desc(edges, checks, slots)
        lam = np.ascontiguousarray(lam, np.float64)
        B, q = lam.shape[0], 1 << m
        hard = np.empty((B, slots), np.int32)
        marg = np.empty((B, slots, q), np.float64)
        conv = np.empty(B, np.int32)
        its = np.empty(B, np.int32)
        self._check(self.h.ref_bp_decode(m, C.byref(cd), B, _p(lam), max_iters, message_floor, int(early_exit), _p(hard),
                                         _p(marg), _p(conv), _p(its)))
        return hard, marg, conv, its

    def sic_decode(self, m: int, edges: np.ndarray, checks: int, slots: int, S: np.ndarray, k: int,
                   max_iters: int = 50, message_floor: float = 1e-30, early_exit: bool = True,
                   cancel_value: float = float("nan")):
        """ura::sic_decode (bp.cpp:349-368) per bin: (grid B x K x L, stage converged, stage iters)."""
        cd, _e = code_desc(edges, checks, slots)
        S = np.ascontiguousarray(S, np.float64)
        B = S.shape[0]
        grid = np.empty((B, k, slots), np.int32)
        sc = np.empty((B, k), np.int32)
        si = np.empty((B, k), np.int32)
        self._check(self.h.ref_sic_decode(m, C.byref(cd), B, k, _p(S), max_iters, message_floor, int(early_exit),
                                          cancel_value, _p(grid), _p(sc), _p(si)))
        return grid, sc, si


    # ---- AMP slot detector (amp.cpp, sim.cpp) --------------------------------------------------
    def amp_make_dicts(self, q: int, n_s: int, slots: int, seed: int) -> np.ndarray:
        """make_dictionaries (sim.cpp:74-80): slots x q x n_s complex."""
        d = np.empty((slots, q, n_s), np.complex128)
        self._check(self.h.ref_amp_make_dicts(q, n_s, slots, C.c_uint64(seed), _p(d)))
        return d

    def amp_observe(self, dicts: np.ndarray, symbols: np.ndarray, p_sym: float, noise_var: float, seed: int) -> np.ndarray:
        """activity_vector + transmit per slot on make_rng(seed): symbols slots x K -> y slots x n_s complex."""
        dicts = np.ascontiguousarray(dicts, np.complex128)
        L, q, n_s = dicts.shape
        sym = np.ascontiguousarray(symbols, np.int32)
        y = np.empty((L, n_s), np.complex128)
        self._check(self.h.ref_amp_observe(q, n_s, L, _p(dicts), sym.shape[1], _p(sym), C.c_double(p_sym),
                                           C.c_double(noise_var), C.c_uint64(seed), _p(y)))
        return y

    def amp_detect_frame(self, dicts: np.ndarray, y: np.ndarray, iters: int = 20, rho_bg: float = 0.03125,
                         sigma_u2: float = 20.0, evidence_floor: float = -40.0) -> np.ndarray:
        """detect_frame (amp.cpp:133-148): S slots x q."""
        dicts = np.ascontiguousarray(dicts, np.complex128)
        L, q, n_s = dicts.shape
        y = np.ascontiguousarray(y, np.complex128)
        S = np.empty((L, q), np.float64)
        self._check(self.h.ref_amp_detect_frame(q, n_s, L, _p(dicts), _p(y), iters, C.c_double(rho_bg),
                                                C.c_double(sigma_u2), C.c_double(evidence_floor), _p(S)))
        return S

    def symbol_power(self, eb_db: float, payload_bits: int, slots: int) -> float:
        f = self.h.ref_symbol_power
        f.restype = C.c_double
        f.argtypes = [C.c_double, C.c_int, C.c_int]
        return f(eb_db, payload_bits, slots)


class RefSession:
    """Decodes through the reference's own engine (ura::run_refinement + MaxProbScorer + remask_pass,
    ref_shim's refine_one) on `threads` host threads, paused between denoiser forwards: advance(n) lets
    every worker run n more forwards and returns when all are parked (bench.py's reference arm)."""

    def __init__(self, ref: "Reference", model: Model, weights: np.ndarray, edges: np.ndarray, checks: int, slots: int,
                 K: int, S: np.ndarray, sched: RevealSchedule, remask: Optional[RemaskConfig], threads: int):
        self.ref = ref
        self._w = np.ascontiguousarray(weights, np.float64)
        self._S = np.ascontiguousarray(S, np.float64)
        self.cd, self._e = code_desc(edges, checks, slots)
        self.n, self.K, self.L = self._S.shape[0], K, slots
        md, sd, rd = model.desc(), sched.desc(), (remask or RemaskConfig()).desc()
        h = C.c_void_p()
        ref._check(ref.h.ref_session_create(C.byref(md), _p(self._w), C.byref(self.cd), K, self.n, _p(self._S),
                                            C.byref(sd), C.byref(rd), threads, C.byref(h)))
        self.h = h

    def advance(self, n: int = 1):
        self.ref._check(self.ref.h.ref_session_advance(self.h, n))

    def status(self):
        f, b = C.c_int64(), C.c_int64()
        grids = np.empty((self.n, self.K, self.L), np.int32)
        done = np.empty(self.n, np.int32)
        self.ref._check(self.ref.h.ref_session_status(self.h, C.byref(f), C.byref(b), _p(grids), _p(done)))
        return {"forwards": f.value, "bins_done": b.value, "grids": grids, "done": done.astype(bool)}

    def close(self):
        if getattr(self, "h", None):
            self.ref.h.ref_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefCli:
    """oracle/_ref/libura_cli.so: the reference's dataset.cpp (with nlohmann/json 3.11.3) and uradec's
    simulate / decode steps composed from the reference library (oracle/ref_cli_shim.cpp)."""
    PATH = os.path.join(_HERE, "_ref", "libura_cli.so")

    def __init__(self):
        from paper_2605_26580_b200 import RunConfigDesc
        self.h = C.CDLL(self.PATH)
        h, P, RC = self.h, C.c_void_p, C.POINTER(RunConfigDesc)
        h.refcli_last_error.restype = C.c_char_p
        for f in ("refcli_config_to_json", "refcli_config_fingerprint"):
            getattr(h, f).argtypes = [RC, C.c_char_p, C.c_int]
        h.refcli_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
        h.refcli_json_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
        h.refcli_simulate.argtypes = [RC, C.c_char_p, C.c_char_p]
        h.refcli_load.argtypes = [C.c_char_p, RC, C.c_char_p, C.c_char_p, C.POINTER(C.c_int), C.c_int, P, P, P, P]
        h.refcli_decode_row.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, P, C.c_int, C.c_int,
                                        C.c_uint64, C.c_int, C.c_char_p, C.c_int]

    @staticmethod
    def available() -> bool:
        return os.path.exists(RefCli.PATH)

    def _check(self, rc):
        if rc == 0:
            return
        msg = self.h.refcli_last_error().decode()
        raise (ValueError if rc == 3 else RuntimeError)(msg)

    def _str(self, fn, *args, cap=4096):
        buf = C.create_string_buffer(cap)
        self._check(fn(*args, buf, cap))
        return buf.value.decode()

    def config_to_json(self, cfg):
        return self._str(self.h.refcli_config_to_json, C.byref(cfg))

    def config_fingerprint(self, cfg):
        return self._str(self.h.refcli_config_fingerprint, C.byref(cfg))

    def format_double(self, x):
        return self._str(self.h.refcli_format_double, float(x))

    def json_double(self, x):
        return self._str(self.h.refcli_json_double, float(x))

    def simulate(self, cfg, dataset_path: str, hfile: str):
        self._check(self.h.refcli_simulate(C.byref(cfg), dataset_path.encode(), hfile.encode()))

    def load(self, path: str) -> dict:
        from paper_2605_26580_b200 import RUN_CONFIG_FIELDS, RunConfigDesc
        cfg = RunConfigDesc()
        fp, hfp, n = C.create_string_buffer(17), C.create_string_buffer(17), C.c_int()
        big = 1 << 14
        self._check(self.h.refcli_load(path.encode(), C.byref(cfg), fp, hfp, C.byref(n), 0, None, None, None, None))
        k, L, q, m = cfg.k, cfg.l, cfg.q, n.value
        seeds, truth = np.empty(m, np.uint64), np.empty((m, k, L), np.int32)
        ev, snr = np.empty((m, L, q), np.float64), np.empty(m, np.float64)
        self._check(self.h.refcli_load(path.encode(), C.byref(cfg), fp, hfp, C.byref(n), m, _p(seeds), _p(truth), _p(ev),
                                       _p(snr)))
        conf = {f: getattr(cfg, f) for f in RUN_CONFIG_FIELDS}
        conf["scale"] = conf["scale"].decode()
        del big
        return {"config": conf, "fingerprint": fp.value.decode(), "h_fingerprint": hfp.value.decode(), "seeds": seeds,
                "truth": truth, "evidence": ev, "snr_db": snr}

    def decode_row(self, dataset: str, hfile: str, decoder: str, scorer: str = "maxprob", steps: int = 0,
                   thresholds=(), latent_dim: int = 128, param_seed: int = 1, f32: bool = True) -> str:
        th = np.ascontiguousarray(thresholds, np.float64)
        return self._str(self.h.refcli_decode_row, dataset.encode(), hfile.encode(), decoder.encode(), scorer.encode(),
                         steps, _p(th) if len(th) else None, len(th), latent_dim, C.c_uint64(param_seed), int(f32))


def derive_seed(master: int, index: int) -> int:
    """seeding.hpp:16-22 (pure-Python restatement, used to name fixture seeds)."""
    M = (1 << 64) - 1

    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    return mix(master ^ mix((index + 0x517CC1B727220A95) & M))
