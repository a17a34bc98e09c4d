"""the reference's dataset format in libcider's host code (csrc/host/dataset.cpp),
pinned against the reference's own dataset.cpp (oracle/_ref/libura_cli.so, built against
nlohmann/json 3.11.3): canonical config JSON and its FNV-1a fingerprint, nlohmann's double layout,
format_double, and load_dataset of reference-written files (bit-identical frames), with the
reference's failure messages. The device decode of a dataset (uradec-gpu) is in test_gpu_parity.py."""
import json
import os
import struct

import numpy as np
import pytest

from oracle.binding import RefCli

pytestmark = pytest.mark.skipif(not RefCli.available(), reason="oracle/_ref/libura_cli.so not built")


@pytest.fixture(scope="module")
def cli():
    return RefCli()


def _doubles(n, seed=0):
    rng = np.random.default_rng(seed)
    vals = [0.0, -0.0, 1.0, -1.0, 10.0, -40.0, 0.1, 1e-4, 1e-5, 9.999e-5, 123456789012345.0, 1e15, 1e16, 2.5e-300,
            1.7976931348623157e308, 5e-324, 3.14159, 1 / 3, 2 / 3, 1e21, 12.5, 0.001]
    vals += list(rng.normal(size=n) * 10.0 ** rng.integers(-20, 20, size=n))
    vals += [float(struct.unpack("<d", rng.bytes(8))[0]) for _ in range(n)]
    vals = [float(v) for v in vals]
    return [v for v in vals if np.isfinite(v)]


def test_json_double_layout_matches_nlohmann(P, cli):
    for x in _doubles(400):
        c = P.run_config(eb_db=x)
        ours = json.loads(P.config_to_json(c).replace("null", "0"))  # structure check
        assert isinstance(ours, dict)
        assert P.config_to_json(c) == cli.config_to_json(c), x


def test_config_json_and_fingerprint_match_reference(P, cli):
    rng = np.random.default_rng(3)
    for i in range(200):
        c = P.run_config(scale=["tiny", "small", "moderate", "large", "x\"y\\z\t"][i % 5], q=int(2 ** rng.integers(1, 9)),
                         l=int(rng.integers(2, 300)), p=int(rng.integers(1, 100)), k=int(rng.integers(1, 9)),
                         n_s=int(rng.integers(1, 64)), eb_db=float(rng.normal() * 20), noise_var=float(rng.random()),
                         amp_iters=int(rng.integers(1, 50)), rho_bg=float(rng.random() - 0.5),
                         sigma_u2=float(rng.normal() * 100), evidence_floor=float(-rng.random() * 100),
                         seed=int(rng.integers(0, 2 ** 63)) * 2 + 1, frames=int(rng.integers(1, 10 ** 6)))
        assert P.config_to_json(c) == cli.config_to_json(c)
        assert P.config_fingerprint(c) == cli.config_fingerprint(c)


def test_format_double_matches_reference(P, cli):
    for x in _doubles(300, seed=7):
        assert P.format_double(x) == cli.format_double(x), x


def test_load_dataset_bit_identical_to_reference(P, cli, tmp_path):
    ds, hf = str(tmp_path / "d.jsonl"), str(tmp_path / "h.txt")
    cfg = P.run_config(frames=12, eb_db=7.5, seed=9)
    cli.simulate(cfg, ds, hf)
    a, b = P.load_dataset(ds), cli.load(ds)
    assert a["config"] == b["config"] and a["fingerprint"] == b["fingerprint"] and a["h_fingerprint"] == b["h_fingerprint"]
    for k in ("seeds", "truth", "evidence", "snr_db"):
        assert np.array_equal(a[k], b[k]), k
    assert a["evidence"].shape == (12, 12, 64) and np.isfinite(a["evidence"]).all()


def test_load_dataset_failures_like_reference(P, cli, tmp_path):
    ds, hf = str(tmp_path / "d.jsonl"), str(tmp_path / "h.txt")
    cli.simulate(P.run_config(frames=3), ds, hf)
    lines = open(ds).read().splitlines()

    def case(name, text):
        p = str(tmp_path / name)
        with open(p, "w") as f:
            f.write(text)
        with pytest.raises(RuntimeError) as ea:
            P.load_dataset(p)
        with pytest.raises(RuntimeError) as eb:
            cli.load(p)
        return str(ea.value), str(eb.value)

    a, b = case("empty.jsonl", "")
    assert a == b == f"load_dataset: empty file {tmp_path / 'empty.jsonl'}"
    a, b = case("nohead.jsonl", "\n".join(lines[1:]) + "\n")
    assert a == b and "missing header record" in a
    h = json.loads(lines[0])
    h["config"]["k"] = 3
    a, b = case("fp.jsonl", json.dumps(h) + "\n" + "\n".join(lines[1:]) + "\n")
    assert a == b and "config fingerprint mismatch" in a
    r = json.loads(lines[1])
    r["config_fp"] = "0" * 16
    a, b = case("ffp.jsonl", lines[0] + "\n" + json.dumps(r) + "\n")
    assert a == b and "frame/config fingerprint mismatch" in a
    r = json.loads(lines[1])
    r["evidence"] = r["evidence"][:-1]
    a, b = case("dims.jsonl", lines[0] + "\n" + json.dumps(r) + "\n")
    assert a == b and "frame dimensions disagree with config" in a
    with pytest.raises(RuntimeError, match="cannot open"):
        P.load_dataset(str(tmp_path / "missing.jsonl"))


def test_file_fingerprint(P, tmp_path):
    import ctypes as C
    p = tmp_path / "x.txt"
    p.write_bytes(b"abc\n")
    buf = C.create_string_buffer(17)
    P._check(P.lib().cider_file_fingerprint(str(p).encode(), buf))
    h = 0xcbf29ce484222325
    for c in b"abc\n":
        h = ((h ^ c) * 0x100000001b3) & (2 ** 64 - 1)
    assert buf.value.decode() == f"{h:016x}"
