"""The ``vc3`` command line (mirrors pkg/tests/test_cli.py).  Argument and
stream-header errors are host-side and run on CPU; everything that computes
is ``-m gpu``."""

import json

import numpy as np
import pytest

from paper_2003_02633_b200 import DEFAULT_LAYOUT
from paper_2003_02633_b200.cli import main
from paper_2003_02633_b200.stream import read_csv, read_stream, write_csv, write_f32, write_stream


def run(capsys, *argv):
    code = main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


# -- CPU ---------------------------------------------------------------------
def test_usage_error_exit_code(capsys):
    for argv in (["analyze", "--domain"], ["no-such-command"], ["bench", "--repeats", "x"]):
        with pytest.raises(SystemExit) as exc:
            main(argv)
        assert exc.value.code == 1


def test_bad_domain_and_grid_are_data_errors(capsys):
    code, _, err = run(capsys, "analyze", "--domain", "torus", "--samples", "10")
    assert code == 2 and "unknown domain" in err
    code, _, err = run(capsys, "misses", "--domain", "shell:1", "--samples", "10")
    assert code == 2 and "shell" in err
    code, _, err = run(capsys, "anisotropy", "--grid", "8by4", "--samples", "10")
    assert code == 2 and "grid" in err


def test_corrupted_stream_is_data_error(golden, tmp_path, capsys):
    packed = tmp_path / "bad.vc3"
    write_stream(packed, golden["cw_17_18_SSS_kat"], DEFAULT_LAYOUT)
    data = bytearray(packed.read_bytes())
    data[:4] = b"XXXX"
    packed.write_bytes(bytes(data))
    code, _, err = run(capsys, "decompress", "--input", str(packed),
                       "--output", str(tmp_path / "x.f32"))
    assert code == 2 and "magic" in err
    packed.write_bytes(bytes(data[:10]))
    code, _, err = run(capsys, "decompress", "--input", str(packed))
    assert code == 2
    code, _, err = run(capsys, "decompress", "--input", str(tmp_path / "missing.vc3"))
    assert code == 2


# -- GPU ---------------------------------------------------------------------
@pytest.mark.gpu
def test_compress_decompress_round_trip_binary(oracle, cuda, tmp_path, capsys):
    v = np.random.default_rng(5).uniform(-1, 1, (100, 3)).astype(np.float32)
    raw, packed, restored = tmp_path / "in.f32", tmp_path / "out.vc3", tmp_path / "back.f32"
    write_f32(raw, v)
    code, _, err = run(capsys, "compress", "--input", str(raw), "--output", str(packed),
                       "--layout", "0,7,22-17-18")
    assert code == 0 and "compressed 100 vectors" in err and "flushed 0, saturated 0" in err
    assert packed.stat().st_size == 20 + 8 * 100
    words, lay = read_stream(packed)
    code, _, _ = run(capsys, "decompress", "--input", str(packed), "--output", str(restored))
    assert code == 0 and restored.stat().st_size == 1200
    back = np.fromfile(restored, dtype="<f4").reshape(-1, 3)
    assert np.array_equal(back.view(np.uint32), oracle.decompress(words, lay).view(np.uint32))
    nv = np.linalg.norm(v.astype(np.float64), axis=1)
    assert (np.linalg.norm(back.astype(np.float64) - v, axis=1) <= 3e-4 * nv + 1e-12).all()


@pytest.mark.gpu
def test_zero_triplet_csv_and_layout_flag(cuda, tmp_path, capsys):
    write_f32(tmp_path / "z.f32", np.zeros((1, 3), np.float32))
    code, _, _ = run(capsys, "compress", "--input", str(tmp_path / "z.f32"),
                     "--output", str(tmp_path / "z.vc3"))
    assert code == 0 and (tmp_path / "z.vc3").stat().st_size == 28
    v = np.random.default_rng(6).uniform(-1, 1, (100, 3)).astype(np.float32)
    write_csv(tmp_path / "in.csv", v)
    code, _, _ = run(capsys, "compress", "--input", str(tmp_path / "in.csv"), "--output",
                     str(tmp_path / "c.vc3"), "--input-format", "csv", "--layout", "0,8,23-16-17")
    assert code == 0
    _, lay = read_stream(tmp_path / "c.vc3")
    assert (lay.exponent_bits, lay.phi_bits, lay.theta_bits, lay.exponent_bias) == (8, 16, 17, 127)
    code, _, _ = run(capsys, "decompress", "--input", str(tmp_path / "c.vc3"), "--output",
                     str(tmp_path / "back.csv"), "--output-format", "csv")
    back = read_csv(tmp_path / "back.csv")
    assert code == 0 and back.shape == (100, 3)
    assert (np.linalg.norm(back - v, axis=1) / np.linalg.norm(v, axis=1)).max() <= 3e-4


@pytest.mark.gpu
def test_studies_json(cuda, capsys):
    code, out, _ = run(capsys, "analyze", "--samples", "20000", "--seed", "1", "--json",
                       "--normalised")
    doc = json.loads(out)
    assert code == 0 and doc["count"] == 20000 and doc["layout"] == "<0,7,22>-17-18"
    assert 5e-6 < doc["mean"] < 1.2e-5
    code, out, _ = run(capsys, "misses", "--samples", "50000", "--seed", "42", "--json")
    doc = json.loads(out)
    assert code == 0 and 0 <= doc["misses_theta"] < 0.01 and 0 <= doc["misses_phi"] < 0.01
    code, out, _ = run(capsys, "compand", "--kind", "cosine", "--samples", "30000", "--json")
    doc = json.loads(out)
    assert code == 0 and doc["mean"] > doc["uniform_mean"]
    code, out, _ = run(capsys, "idempotence", "--samples", "1000", "--seed", "3",
                       "--policy", "theta=D,phi=D,quant=D", "--json")
    assert code == 0 and json.loads(out)["word_miss_fraction"] == 0.0


@pytest.mark.gpu
def test_anisotropy_and_sweep_text(cuda, capsys):
    code, out, _ = run(capsys, "anisotropy", "--samples", "30000", "--grid", "8x4")
    lines = out.strip().splitlines()
    assert code == 0 and lines[0] == "theta_cell,phi_cell,mean_error" and len(lines) == 33
    i, j, m = lines[1].split(",")
    assert 0 <= int(i) < 8 and 0 <= int(j) < 4 and float(m) > 0
    code, out, _ = run(capsys, "sweep", "--bits", "35", "--splits", "131072,196608",
                       "--samples", "20000")
    assert code == 0 and out.count("n_phi_max+1") == 2


@pytest.mark.gpu
def test_bench_csv_and_json(cuda, capsys):
    code, out, _ = run(capsys, "bench", "--sizes", "4096,8192", "--repeats", "3")
    lines = out.strip().splitlines()
    assert code == 0 and lines[0] == "n,time_raw_ns,time_comp_ns,speedup,bytes_ratio"
    assert len(lines) == 3 and all(line.endswith(",1.5") for line in lines[1:])
    code, out, _ = run(capsys, "bench", "--sizes", "4096,16777216", "--repeats", "3", "--json")
    doc = json.loads(out)
    assert code == 0 and doc["llc_bytes"] > 50 << 20 and doc["knee_elements"] == 4096
    big = doc["rows"][1]
    assert big["gvec_s_compressed"] > 10 and big["gbs_raw"] > 1000
