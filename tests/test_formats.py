"""the reference's parity-check file format (ldpc.cpp:197-226), both directions
against the compiled reference (CPU only)."""
import os

import numpy as np
import pytest


def test_parity_file_round_trips_with_the_reference(P, reference, tmp_path):
    for name in ("c1", "c3", "c4"):
        wl = P.configs()[name].workload
        e = wl.code()
        ours, theirs = str(tmp_path / f"{name}_ours.txt"), str(tmp_path / f"{name}_ref.txt")
        P.save_parity_file(ours, e, wl.checks, wl.slots, 1 << wl.m, wl.col_weight, 0, 1)
        reference.save_parity_file(theirs, wl.m, e, wl.checks, wl.slots, wl.col_weight, 0, 1)
        assert open(ours).read() == open(theirs).read()          # byte-identical files
        a, b = P.load_parity_file(theirs), reference.load_parity_file(ours)
        for k in ("checks", "slots", "q", "col_weight", "prim_poly", "seed"):
            assert a[k] == b[k]
        assert np.array_equal(a["edges"], b["edges"]) and np.array_equal(a["edges"], e)


def test_parity_file_errors_like_the_reference(P, tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("8 16 16 3\n")
    with pytest.raises(RuntimeError, match="load_parity_file: malformed header"):
        P.load_parity_file(str(bad))
    bad.write_text("2 4 16 3 19 1\n0 0 1\n0 1 x\n")
    with pytest.raises(RuntimeError, match="load_parity_file: malformed entry line"):
        P.load_parity_file(str(bad))
    bad.write_text("2 4 16 3 19 1\n0 0 1\n5 1 3\n")
    with pytest.raises(RuntimeError, match="load_parity_file: invalid matrix"):
        P.load_parity_file(str(bad))
    with pytest.raises(RuntimeError, match="cannot open"):
        P.load_parity_file(str(tmp_path / "missing.txt"))
