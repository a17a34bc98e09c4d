"""The C-ABI library: loads, exports every symbol include/cider.h declares, validates its inputs
on the host, and fails loudly (no CPU fallback) when there is no GPU."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(P):
    lib_path = P.LIB_PATH
    assert os.path.exists(lib_path)
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    declared = P.exported_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    h = C.CDLL(lib_path)
    for s in declared:
        getattr(h, s)


def test_header_cites_reference_interfaces():
    hdr = open(os.path.join(ROOT, "include", "cider.h")).read()
    for cite in ["denoiser.hpp:109-114", "refine.hpp:60-62", "refine.hpp:104-107", "denoiser.cpp:41-69"]:
        assert cite in hdr


def test_weights_count_layout(P):
    m = P.Model(m=6, dim=32, hidden=48, layers=3, heads=4)
    q, D, H, N = 64, 32, 48, 3
    per = (H * 2 * D + H + D * H + D) * 2 + (H * D + H + D * H + D)
    assert P.weights_count(m) == (q + 1) * D + 2 * q * D + N * per + N * (D + D * D)


def test_invalid_model_rejected_on_host(P):
    with pytest.raises(ValueError):
        P.weights_init(P.Model(m=9, dim=8, hidden=8), 1)
    with pytest.raises(ValueError):
        P.weights_init(P.Model(m=4, dim=10, hidden=8, heads=4), 1)


def test_no_cpu_fallback_without_gpu(P):
    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    m = P.Model.ref_exact(4, 16)
    wl = P.configs()["c1"].workload
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.Context(m, P.weights_init(m, 1), wl.code(), wl.checks, wl.slots)


def test_invalid_code_rejected_before_any_device_work(P):
    m = P.Model.ref_exact(4, 16)
    bad = np.array([[0, 0, 3], [0, 0, 5]], np.int32)  # duplicate (check, slot)
    with pytest.raises(ValueError, match="duplicate"):
        P.Context(m, P.weights_init(m, 1), bad, 1, 4)
    zero = np.array([[0, 1, 0]], np.int32)
    with pytest.raises(ValueError, match="nonzero"):
        P.Context(m, P.weights_init(m, 1), zero, 1, 4)


def test_dense_code_construction_is_defined(P):
    """3 L / P > P + 1: every free check's degree exceeds the reference's scan start (ldpc.cpp:103), where its
    candidate list is empty and the draw undefined; the product builds a valid balanced code instead."""
    for m, slots, checks in [(5, 9, 4), (3, 9, 3), (6, 20, 3), (4, 30, 5)]:
        wl = P.Workload(m=m, slots=slots, checks=checks, k=2, snr_db=3.0)
        e = wl.code()
        assert e.shape == (slots * wl.col_weight, 3)
        assert np.all((e[:, 2] >= 1) & (e[:, 2] < (1 << m)))
        for l in range(slots):
            assert len(set(e[e[:, 1] == l, 0])) == wl.col_weight  # distinct checks per slot
        deg = np.bincount(e[:, 0], minlength=checks)
        assert deg.max() - deg.min() <= 1
        truth, S = wl.bins(e, 0, 2)  # systematic form exists (full rank), codewords satisfy H
        assert truth.shape == (2, 2, slots) and np.isfinite(S).all()
