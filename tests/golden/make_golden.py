"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libura_ref.so, built by
oracle/Makefile from /root/reference/proj/src). Run in the build container (where /root/reference
exists); the fixtures are committed so the GPU box, which has no reference tree, can still pin the
oracle restatement and the product's host code.

    python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_2605_26580_b200 as P  # noqa: E402
from oracle.binding import Reference, derive_seed  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Reference()
    out = {}
    # (1) DenoiserParams::random_init(64, 32, 7) and (16, 64, 1)
    for q, d, s in [(64, 32, 7), (16, 64, 1)]:
        w = ref.random_init(q, d, s)
        out[f"init_q{q}_d{d}_s{s}_sha"] = np.array(sha(w))
        out[f"init_q{q}_d{d}_s{s}_head"] = w[:32]
        out[f"init_q{q}_d{d}_s{s}_tail"] = w[-32:]
    # (2) build_random_ldpc + sample_codewords for the BASELINE configs (uradec.cpp:45-54 seeds)
    for name, c in P.configs().items():
        if name == "c5":
            continue
        wl = c.workload
        e = ref.build_ldpc(wl.m, wl.slots, wl.checks, wl.col_weight, derive_seed(0, 1))
        out[f"{name}_edges"] = e
        out[f"{name}_codewords"] = np.stack(
            [ref.sample_codewords(wl.m, e, wl.checks, wl.slots, wl.k, derive_seed(0, 16 + b)) for b in range(3)])
    # (3) denoiser forwards + refinement runs on c1-shaped inputs
    wl = P.configs()["c1"].workload
    e = out["c1_edges"]
    truth, S = wl.bins(e, 0, 2)
    S64 = S.astype(np.float64)
    out["c1_S"] = S
    rng = np.random.default_rng(2024)
    X = rng.integers(-1, 16, size=(2, 16)).astype(np.int32)
    out["c1_X"] = X
    models = {
        "refexact": P.Model.ref_exact(4, 64),
        "stacked": P.Model(m=4, dim=64, hidden=128, layers=2, heads=0),
        "attn": P.Model(m=4, dim=64, hidden=128, layers=2, heads=4),
    }
    for tag, m in models.items():
        w = P.weights_init(m, 1).astype(np.float64)
        out[f"{tag}_weights_sha"] = np.array(sha(P.weights_init(m, 1)))
        lg, inc = ref.denoise(m, w, e, wl.checks, wl.slots, X, S64[0], want_incoming=True)
        out[f"{tag}_logits"] = lg
        out[f"{tag}_incoming"] = inc
        r = ref.refine(m, w, e, wl.checks, wl.slots, S64, 2, P.RevealSchedule(steps=4), want_final_logits=True)
        out[f"{tag}_grid"] = r["grid"]
        out[f"{tag}_final_logits"] = r["final_logits"]
        out[f"{tag}_first"] = r["first_reveals"]
    # (4) remasking: K=8, threshold schedule (refine.cpp:277-292) and the rank adapter
    wl8 = P.Workload(m=4, slots=16, checks=8, k=8, snr_db=4.0, p_erase=0.1, p_false=0.1)
    e8 = out["c1_edges"]
    _, S8 = wl8.bins(e8, 0, 2)
    out["k8_S"] = S8
    m8 = P.Model.ref_exact(4, 32)
    w8 = P.weights_init(m8, 3).astype(np.float64)
    for tag, rm in [("thr", P.RemaskConfig(thresholds=(0.3, 0.2, 0.1))), ("rank", P.RemaskConfig(rank_fraction=0.25))]:
        r = ref.refine(m8, w8, e8, 8, 16, S8.astype(np.float64), 8, P.RevealSchedule(steps=6), rm, want_final_logits=True)
        for k, v in r.items():
            out[f"k8_{tag}_{k}"] = v
    # (5) reveal_step with ties (identical rows -> exact kappa ties, refine.cpp:115-119)
    lg = rng.normal(size=(3, 12, 64))
    lg[2] = lg[1]
    Xr = np.full((3, 12), -1, np.int32)
    Xr[0, :3] = [4, 5, 6]
    out["reveal_logits"] = lg
    out["reveal_X"] = Xr
    out["reveal_first"] = ref.reveal_step(Xr, lg, 0, 1.0, True)
    out["reveal_t20"] = ref.reveal_step(Xr, lg, 20, 0.7, False)
    # (6) WHT-domain GF(Q) check update (bp.cpp:128-149) vs the direct O(Q^2) one
    for m, d in [(4, 3), (6, 5)]:
        q = 1 << m
        inc = rng.random((d, q))
        inc /= inc.sum(1, keepdims=True)
        cf = rng.integers(1, q, size=d).astype(np.int32)
        out[f"wht_m{m}_in"] = inc
        out[f"wht_m{m}_coef"] = cf
        out[f"wht_m{m}_out"] = ref.check_update_wht(m, inc, cf, 3)
        out[f"wht_m{m}_direct"] = ref.check_update_direct(m, inc, cf, 3)
    # (7) SER/CER with the lexicographic Hungarian tie rule (metrics.cpp:79-145)
    t = rng.integers(0, 4, size=(20, 4, 6)).astype(np.int32)
    p = t.copy()
    p[:, :, :3] = rng.integers(0, 4, size=(20, 4, 3))
    p = p[:, rng.permutation(4)]
    out["ser_truth"], out["ser_pred"] = t, p
    out["ser_ref"] = np.array([ref.ser_cer(t[i], p[i]) for i in range(20)])
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_vectors.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
