"""Decision parity at the BASELINE shapes (VERDICT r1 "next" 1).

* BF16 (the throughput mode): the FULL config models (c3/c5: N=6, D=256, H=1024, 8 heads, K=8,
  Q=256, T=16 + rank-25% remask; c2; c4) decode a batch large enough that every CTA pair of the
  persistent 2-SM MLP / grouped-GEMM kernels runs many tiles, with probe bins at the first, last and
  late-tile positions. Every forward of the probe bins is re-run on the CPU oracle with the device's
  own input grid (teacher forcing) and every device decision — reveal sets, revealed symbols, final
  argmax, remask rows — is re-derived from the oracle's logits. Logits within BF16_TOL; every decision
  that differs (a flip) must sit at an oracle margin the measured logit error can cross
  (tests/teacher_forced.py); carried sites bit-identical.
* FP32 (the parity mode): full decodes of the config models (c2 16 bins, c3 4 bins, c4 2 bins)
  against oracle.refine: identical grids, remask rows / steps / masks, final logits within 1e-3.

Measured numbers go to the session's parity report ($CIDER_PARITY_REPORT).
"""
import numpy as np
import pytest

from oracle import teacher_forced as tf
from conftest import rel_err

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2   # logits, relative to max |logit| of the bin and record
FP32_TOL = 1e-3


def _setup(P, name, precision=None, nb=None):
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    if precision is not None:
        model = P.Model(**{**model.__dict__, "precision": precision})
    e = wl.code()
    w = P.weights_init(model, 1)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    truth, S = wl.bins(e, 0, nb or cfg.bins)
    return cfg, wl, model, e, w, ctx, truth, S


@pytest.mark.parametrize("name,nb,probe", [
    # c3 / c5: 512 bins -> 2048 aggregator pair-tiles over 74 CTA pairs (>= 27 tiles per pair);
    # bins >= 148 are past the gate / fusion kernels' 4th tile round
    ("c3", 512, [0, 1, 149, 255, 256, 300, 510, 511]),
    ("c2", 2048, [0, 777, 1500, 2047]),
    ("c4", 160, [0, 159]),
])
def test_bf16_teacher_forced_decisions(P, oracle, parity_report, name, nb, probe):
    cfg, wl, model, e, w, ctx, truth, S = _setup(P, name, nb=nb)
    S[300 % nb] = S[0]  # one replica: a bin's decode must not depend on its batch position
    sched = P.RevealSchedule(steps=cfg.steps)
    grid, st, det = tf.teacher_forced(P, oracle, ctx, model, P.model_weights_as_run(model, w), e, wl, S, sched,
                                      cfg.remask, probe)
    # the probe run is the plain device decode: same grids as cider_refine
    assert np.array_equal(grid, ctx.refine(S, wl.k, sched, cfg.remask))
    assert np.array_equal(grid[300 % nb], grid[0])
    rep = st.as_dict()
    rep.update(bins=nb, probe_bins=probe, per_bin_rel_err=det["per_bin_rel_err"],
               ser_device_probe=P.ser_cer(truth[probe], grid[probe])[0])
    parity_report[f"bf16_teacher_forced_{name}"] = rep
    print(name, rep)
    assert st.max_rel_err < BF16_TOL, rep
    assert st.carry_mismatch == 0, rep
    assert not st.unexplained, st.unexplained[:10]
    assert st.agreement > 0.97, rep


@pytest.mark.parametrize("name,nb", [("c2", 16), ("c3", 4), ("c4", 2)])
def test_fp32_full_decode_identical(P, oracle, parity_report, name, nb):
    cfg, wl, model, e, w, ctx, truth, S = _setup(P, name, precision=P.FP32, nb=nb)
    sched = P.RevealSchedule(steps=cfg.steps)
    grid, fl, tr = ctx.refine(S, wl.k, sched, cfg.remask, want_final_logits=True, want_trace=True)
    wr = P.model_weights_as_run(model, w)
    ro = oracle.refine(model, wr, e, wl.checks, wl.slots, S.astype(np.float64), wl.k, sched, cfg.remask,
                       want_final_logits=True)
    err = rel_err(fl, ro["final_logits"])
    same = [bool(np.array_equal(grid[b], ro["grid"][b])) for b in range(nb)]
    rep = {"bins": nb, "final_logits_rel_err": err, "identical_grids": int(sum(same)),
           "ser_device": P.ser_cer(truth, grid)[0], "ser_oracle": P.ser_cer(truth, ro["grid"])[0]}
    parity_report[f"fp32_full_decode_{name}"] = rep
    print(name, rep)
    assert err < FP32_TOL
    assert all(same), rep
    assert np.array_equal(tr["first_reveals"], ro["first_reveals"])
    assert np.array_equal(tr["remask_rows"], ro["remask_rows"])
    assert np.array_equal(tr["remask_steps"], ro["remask_steps"])
    assert np.array_equal(tr["remask_mask"], ro["remask_mask"])


def test_fp32_probe_records_match_oracle_trajectory(P, oracle):
    """The probe's record stream (cider_refine_probe) in FP32 mode is the oracle's own trajectory:
    identical input grids for every forward, logits within 1e-3, identical pass outputs."""
    wl = P.Workload(m=6, slots=16, checks=8, k=4, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=6, dim=64, hidden=128, layers=2, heads=4, precision=P.FP32)
    e = wl.code()
    w = P.weights_init(model, 2)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 6)
    sched = P.RevealSchedule(steps=6)
    rm = P.RemaskConfig(rank_fraction=0.5)
    grid, meta, X, lg = ctx.refine_probe(S, wl.k, sched, rm, probe_bins=[1, 5])
    wr = P.model_weights_as_run(model, w)
    for i, b in enumerate([1, 5]):
        m2, X2, lg2, g2 = tf.oracle_trajectory(oracle, model, wr, e, wl, S[b], sched, k_low=2)
        assert np.array_equal(meta, m2)
        assert np.array_equal(X[i], X2)
        fwd = meta[:, 3] < 2
        assert rel_err(lg[i][fwd], lg2[fwd]) < FP32_TOL
        assert np.array_equal(grid[b], g2)


def test_trace_records_like_refine_trace(P, oracle):
    """cider_trace's RefineTrace fields (refine.hpp:48-54): per-pass first-step counts, the most recent
    pass's per-step reveal counts and first-step sites — recomputed from the probe's record stream —
    also with first_reveal = False (the t = 1 count is still recorded, as the reference does)."""
    wl = P.Workload(m=4, slots=16, checks=8, k=4, snr_db=4.0)
    model = P.Model(m=4, dim=32, hidden=64, layers=1, heads=2, precision=P.FP32)
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 3)
    for sched in (P.RevealSchedule(steps=5), P.RevealSchedule(steps=5, first_reveal=False)):
        rm = P.RemaskConfig(rank_fraction=0.5)
        grid, tr = ctx.refine(S, wl.k, sched, rm, want_trace=True)
        _, meta, X, _ = ctx.refine_probe(S, wl.k, sched, rm, probe_bins=[0, 1, 2], want_logits=False)
        for b in range(3):
            starts = [r for r in range(len(meta)) if meta[r][3] == 0 and meta[r][1] == 1]
            firsts = [int(((X[b][r] == -1) & (X[b][r + 1] != -1)).sum()) for r in starts]
            assert tr["n_passes"][b] == len(starts) == 2
            assert list(tr["pass_first_reveals"][b][:2]) == firsts
            assert tr["first_reveals"][b] == firsts[0]
            last = starts[-1]
            T = int(meta[last][2])
            counts = [int(((X[b][r] == -1) & (X[b][r + 1] != -1)).sum()) for r in range(last, last + T)]
            assert tr["n_reveal_counts"][b] == T and T >= 2  # (T = 1 would add the residual forcing)
            assert list(tr["reveal_counts"][b][:T]) == counts
            sites = (X[b][last] == -1) & (X[b][last + 1] != -1)
            if T > 1:
                assert np.array_equal(tr["first_step_sites"][b].astype(bool), sites)


def test_graph_replay_respects_final_logits_request(P):
    """a refinement graph captured without final logits must not be replayed for a
    call that asks for them (the key names the final-logits buffer). Alternate both kinds of call on
    one context at one batch size: every final-logits result is the same."""
    wl = P.Workload(m=4, slots=16, checks=8, k=3, snr_db=4.0)
    model = P.Model(m=4, dim=32, hidden=64, layers=1, heads=2, precision=P.FP32)
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 5)
    _, S2 = wl.bins(e, 50, 5)
    sched = P.RevealSchedule(steps=4)
    ref_g, ref_fl = ctx.refine(S, 3, sched, want_final_logits=True)
    for i in range(3):
        g2 = ctx.refine(S2, 3, sched)            # eager, then captured, then replayed
        g, fl = ctx.refine(S, 3, sched, want_final_logits=True)
        assert np.array_equal(g, ref_g) and np.array_equal(fl, ref_fl), i
        assert g2.shape == g.shape


@pytest.mark.parametrize("L,K", [(1024, 8), (1100, 16)])
def test_large_grids_reveal(P, oracle, L, K):
    """reveal over K*L sites beyond the old 4096-key shared array — 8192 sites (dynamic
    shared memory) and 17600 sites (global-memory key slices) — equals the oracle."""
    wl = P.Workload(m=4, slots=L, checks=L // 2, k=K, snr_db=6.0)
    model = P.Model(m=4, dim=32, hidden=32, layers=1, precision=P.FP32)
    e = wl.code()
    w = P.weights_init(model, 1)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    _, S = wl.bins(e, 0, 2)
    sched = P.RevealSchedule(steps=3)
    g, tr = ctx.refine(S, K, sched, want_trace=True)
    ro = oracle.refine(model, P.model_weights_as_run(model, w), e, wl.checks, wl.slots, S.astype(np.float64), K, sched)
    assert np.array_equal(g, ro["grid"])
    assert np.array_equal(tr["first_reveals"], ro["first_reveals"])


def test_nccl_world1_gather_and_pack(P):
    """cider_nccl_unique_id / init / allgather at world 1 (the gather bench.py closes its timed region
    with) and the uint8 packing of decoded grids."""
    import ctypes as C
    lib = P.lib()
    wl = P.Workload(m=4, slots=16, checks=8, k=3, snr_db=4.0)
    model = P.Model(m=4, dim=32, hidden=32, layers=1, precision=P.FP32)
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    uid = C.create_string_buffer(128)
    P._check(lib.cider_nccl_unique_id(uid))
    P._check(lib.cider_nccl_init(ctx.h, uid.raw, 0, 1))
    g = np.random.default_rng(0).integers(0, 16, size=(5, 3, 16)).astype(np.int32)
    dg, du, dr = C.c_void_p(), C.c_void_p(), C.c_void_p()
    for p, n in ((dg, g.nbytes), (du, g.size), (dr, g.size)):
        P._check(lib.cider_device_alloc(ctx.h, n, C.byref(p)))
    P._check(lib.cider_memcpy_h2d(ctx.h, dg, g.ctypes.data_as(C.c_void_p), g.nbytes))
    P._check(lib.cider_grid_pack_u8(ctx.h, dg, du, g.size))
    P._check(lib.cider_nccl_allgather(ctx.h, du, dr, g.size))
    out = np.empty(g.size, np.uint8)
    P._check(lib.cider_memcpy_d2h(ctx.h, out.ctypes.data_as(C.c_void_p), dr, g.size))
    P._check(lib.cider_synchronize(ctx.h))
    assert np.array_equal(out.reshape(g.shape).astype(np.int32), g)


def test_bench_line_small(P):
    """bench.py end to end on a small c2 batch: one JSON line with the gather verified, launches counted,
    the roofline and e2e keys present."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "c2", "--steps", "2", "--warmup", "1",
                        "--bins-per-step", "256", "--no-cpu-baseline", "--no-parity"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["gpu_launches"] > 0 and line["value"] > 0
    assert line["nccl_gather"]["checksums_match"] is True, line["nccl_gather"]
    assert {"roofline", "e2e", "clocks"} <= set(line)


def test_remask_pass_caller_confidences_and_scorer(P, oracle):
    """cider_remask_pass (ura::remask_pass with caller confidences) vs the oracle in FP32: identical grids,
    bins without a low row untouched; and the reference's stage loop driven by a pluggable scorer
    (run_with_remasking_scored) with MaxProbScorer equals the built-in threshold remasking."""
    wl = P.Workload(m=6, slots=16, checks=8, k=4, snr_db=4.0, p_erase=0.1, p_false=0.1)
    model = P.Model(m=6, dim=64, hidden=96, layers=2, heads=2, precision=P.FP32)
    e = wl.code()
    w = P.weights_init(model, 3)
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    wr = P.model_weights_as_run(model, w)
    _, S = wl.bins(e, 0, 6)
    sched = P.RevealSchedule(steps=5)
    g0 = ctx.refine(S, wl.k, sched)
    conf = np.random.default_rng(1).random((6, wl.k))
    conf[2] = 0.99  # no low row
    g, fl = ctx.remask_pass(S, g0, conf, 0.5, sched, want_final_logits=True)
    go, flo = oracle.remask_pass(model, wr, e, wl.checks, wl.slots, S.astype(np.float64), g0, conf, 0.5, sched)
    assert np.array_equal(g, go)
    assert np.array_equal(g[2], g0[2]) and np.isnan(fl[2]).all()
    has = ~np.isnan(flo[:, 0, 0, 0])
    assert rel_err(fl[has], flo[has]) < FP32_TOL
    den = P.StructuredDenoiser(ctx)
    thr = (0.6, 0.3)
    a = P.run_with_remasking_scored(den, P.MaxProbScorer(), S, sched, thr, wl.k)
    b = ctx.refine(S, wl.k, sched, P.RemaskConfig(thresholds=thr))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("decoder,scorer,thr,k", [("refine-structured", "maxprob", (), 2),
                                                  ("refine-structured", "maxprob", (0.9, 0.6), 3),
                                                  ("refine-structured", "oracle", (0.9, 0.5), 3),
                                                  ("sic-bp", "maxprob", (), 3)])
def test_uradec_gpu_decode_csv_matches_reference(P, tmp_path, decoder, scorer, thr, k):
    """`uradec-gpu decode` (csrc/tools/uradec_gpu.cpp, C ABI only) on a dataset and parity
    file written by the reference's own code writes the reference's CSV: the same preamble, header and
    row (every column but ms_per_sample) as uradec decode's restated steps over the reference library
    (oracle/ref_cli_shim.cpp; FP32 inputs, the values the device's parity mode computes with)."""
    import os
    import subprocess
    from oracle.binding import RefCli
    if not RefCli.available():
        pytest.skip("oracle/_ref/libura_cli.so not built")
    cli = RefCli()
    ds, hf, out = str(tmp_path / "d.jsonl"), str(tmp_path / "h.txt"), str(tmp_path / "r.csv")
    cli.simulate(P.run_config(frames=16, k=k, eb_db=9.0, seed=5), ds, hf)
    exe = os.path.join(os.path.dirname(P.LIB_PATH), "uradec-gpu")
    cmd = [exe, "decode", "--dataset", ds, "--hfile", hf, "--decoder", decoder, "--scorer", scorer, "--out", out]
    if thr:
        cmd += ["--remask-thresholds", ",".join(str(t) for t in thr)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = open(out).read().splitlines()
    cfg_json = cli.config_to_json(P.run_config(frames=16, k=k, eb_db=9.0, seed=5))
    assert lines[0] == "# uradec 0.1.0" and lines[1] == "# config: " + cfg_json
    assert lines[2].startswith("decoder,backend,scale,q,l,p,k,eb_db,snr_db,seed,samples,ser,cer,ms_per_sample")
    ours = lines[3].split(",")
    ref = cli.decode_row(ds, hf, decoder, scorer, 0, thr, f32=True).split(",")
    ours[13] = ref[13] = "-"
    assert ours == ref


@pytest.mark.parametrize("name", ["c3", "c2", "c4"])
def test_guard_bands_intact_after_the_kernel_set(P, name):
    """Out-of-bounds write check for the device kernels (compute-sanitizer is closed on the GPU pool):
    every workspace buffer gets 64 KB 0xA5 guard bands, the config's full kernel set runs (eager and
    graph-replayed refinement with remasking, a forward with messages), and no band byte may change;
    the positive control (a byte poked past a buffer's end) must be reported."""
    cfg = P.configs()[name]
    wl, model = cfg.workload, cfg.model
    e = wl.code()
    ctx = P.Context(model, P.weights_init(model, 1), e, wl.checks, wl.slots)
    ctx.set_debug_guard(65536)
    nb = 40 if name != "c2" else 300
    _, S = wl.bins(e, 0, nb)
    sched = P.RevealSchedule(steps=3)
    for _ in range(3):  # eager, capture, replay
        ctx.refine(S, wl.k, sched, P.RemaskConfig(rank_fraction=0.25))
    X = np.where(np.random.default_rng(1).random((nb, wl.k, wl.slots)) < 0.5, 3, -1).astype(np.int32)
    ctx.denoise(X, S, want_incoming=True)
    ctx.refine(S, wl.k, sched, P.RemaskConfig(thresholds=(0.9, 0.5)), want_trace=True)
    bad, msg = ctx.debug_check()
    assert bad == 0, msg
    import ctypes as C
    P._check(P.lib().cider_debug_poke(ctx.h, b"Nn" if name != "c2" else b"X", 100))
    bad, msg = ctx.debug_check()
    assert bad == 1 and "overwritten" in msg, msg
