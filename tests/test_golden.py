"""The CPU oracle restatement and the product's host code against the committed reference vectors
(tests/golden/reference_vectors.npz, produced from the reference itself by make_golden.py)."""
import hashlib
import os

import numpy as np
import pytest

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("q,d,s", [(64, 32, 7), (16, 64, 1)])
def test_weight_init_matches_random_init(P, q, d, s):
    """cider_weights_init_f64 == DenoiserParams::random_init bit for bit (denoiser.cpp:41-69)."""
    m = P.Model.ref_exact(q.bit_length() - 1, d)
    w = P.weights_init(m, s, f64=True)
    assert sha(w) == str(G[f"init_q{q}_d{d}_s{s}_sha"])
    assert np.array_equal(w[:32], G[f"init_q{q}_d{d}_s{s}_head"])


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_code_and_codewords_match_reference(P, name):
    """build_random_ldpc / sample_codewords replayed on the host (ldpc.cpp:80-195, uradec.cpp:45-54)."""
    wl = P.configs()[name].workload
    e = wl.code()
    assert np.array_equal(e, G[f"{name}_edges"])
    truth, S = wl.bins(e, 0, 3)
    assert np.array_equal(truth, G[f"{name}_codewords"])
    # the evidence rows are log-softmax normalised
    assert np.allclose(np.exp(S.astype(np.float64)).sum(-1), 1.0, atol=1e-5)


@pytest.mark.parametrize("tag", ["refexact", "stacked", "attn"])
def test_oracle_denoise_matches_reference_vectors(P, oracle, tag):
    models = {"refexact": P.Model.ref_exact(4, 64), "stacked": P.Model(m=4, dim=64, hidden=128, layers=2),
              "attn": P.Model(m=4, dim=64, hidden=128, layers=2, heads=4)}
    m = models[tag]
    w32 = P.weights_init(m, 1)
    assert sha(w32) == str(G[f"{tag}_weights_sha"])
    wl = P.configs()["c1"].workload
    lg, inc = oracle.denoise(m, w32.astype(np.float64), G["c1_edges"], wl.checks, wl.slots, G["c1_X"],
                             G["c1_S"][0].astype(np.float64), want_incoming=True)
    # same fp64 operation order and libm as the reference: bit-exact
    assert np.array_equal(lg, G[f"{tag}_logits"])
    assert np.array_equal(inc, G[f"{tag}_incoming"])


@pytest.mark.parametrize("tag", ["refexact", "stacked", "attn"])
def test_oracle_refine_matches_reference_vectors(P, oracle, tag):
    models = {"refexact": P.Model.ref_exact(4, 64), "stacked": P.Model(m=4, dim=64, hidden=128, layers=2),
              "attn": P.Model(m=4, dim=64, hidden=128, layers=2, heads=4)}
    m = models[tag]
    w = P.weights_init(m, 1).astype(np.float64)
    wl = P.configs()["c1"].workload
    r = oracle.refine(m, w, G["c1_edges"], wl.checks, wl.slots, G["c1_S"].astype(np.float64), 2,
                      P.RevealSchedule(steps=4), want_final_logits=True)
    assert np.array_equal(r["grid"], G[f"{tag}_grid"])
    assert np.array_equal(r["final_logits"], G[f"{tag}_final_logits"])
    assert np.array_equal(r["first_reveals"], G[f"{tag}_first"])


@pytest.mark.parametrize("tag", ["thr", "rank"])
def test_oracle_remask_matches_reference_vectors(P, oracle, tag):
    rm = P.RemaskConfig(thresholds=(0.3, 0.2, 0.1)) if tag == "thr" else P.RemaskConfig(rank_fraction=0.25)
    m = P.Model.ref_exact(4, 32)
    w = P.weights_init(m, 3).astype(np.float64)
    r = oracle.refine(m, w, G["c1_edges"], 8, 16, G["k8_S"].astype(np.float64), 8, P.RevealSchedule(steps=6), rm,
                      want_final_logits=True)
    for k in ["grid", "final_logits", "first_reveals", "remask_rows", "remask_steps", "remask_mask"]:
        assert np.array_equal(r[k], G[f"k8_{tag}_{k}"]), k


def test_oracle_reveal_step_ties(oracle):
    lg, X = G["reveal_logits"], G["reveal_X"]
    assert np.array_equal(oracle.reveal_step(X, lg, 0, 1.0, True), G["reveal_first"])
    assert np.array_equal(oracle.reveal_step(X, lg, 20, 0.7, False), G["reveal_t20"])


@pytest.mark.parametrize("m", [4, 6])
def test_oracle_wht_check_update(oracle, m):
    out = oracle.check_update_wht(m, G[f"wht_m{m}_in"], G[f"wht_m{m}_coef"], 3)
    assert np.array_equal(out, G[f"wht_m{m}_out"])
    assert np.abs(out - G[f"wht_m{m}_direct"]).max() < 1e-8  # test_bp.cpp:145-168 tolerance


def test_ser_cer_matches_reference(P):
    t, p = G["ser_truth"], G["ser_pred"]
    for i in range(t.shape[0]):
        s, c = P.ser_cer(t[i], p[i])
        assert s == pytest.approx(G["ser_ref"][i][0], abs=1e-12)
        assert c == pytest.approx(G["ser_ref"][i][1], abs=1e-12)
