"""IBMI1 / CSV files (reference matio.py semantics) and the CLI's host logic."""

import numpy as np
import pytest

from paper_2502_06377_b200 import IoError, matio
from paper_2502_06377_b200.cli import _config, _parser, _partition, main


def test_ibmi1_layout_is_frozen(tmp_path):
    a = np.arange(6, dtype=np.float64).reshape(2, 3) / 7.0
    f = tmp_path / "m.ibmi"
    matio.save_ibmi(f, a)
    raw = f.read_bytes()
    assert raw[:8] == b"IBMI1\x00\x00\x00"
    assert np.frombuffer(raw[8:24], dtype="<u8").tolist() == [2, 3]
    assert np.array_equal(np.frombuffer(raw[24:], dtype="<f8"), a.ravel())
    assert np.array_equal(matio.load_ibmi(f), a)
    assert matio.read_header(f) == (2, 3)


def test_ibmi1_errors(tmp_path):
    f = tmp_path / "bad.ibmi"
    f.write_bytes(b"NOPE0000" + b"\0" * 16)
    with pytest.raises(IoError):
        matio.load_ibmi(f)
    g = tmp_path / "short.ibmi"
    matio.save_ibmi(g, np.eye(3))
    g.write_bytes(g.read_bytes()[:-8])
    with pytest.raises(IoError):
        matio.load_ibmi(g)


def test_csv_roundtrip_and_dispatch(tmp_path):
    a = np.random.default_rng(0).standard_normal((4, 5))
    f = tmp_path / "m.csv"
    matio.save_matrix(f, a)
    assert np.array_equal(matio.load_matrix(f), a)        # repr() keeps every bit
    g = tmp_path / "m.bin"
    matio.save_matrix(g, a)
    assert np.array_equal(matio.load_matrix(g), a)


def test_cli_config_and_partition_parsing():
    ap = _parser()
    args = ap.parse_args(["invert", "--in", "x.ibmi", "--guess", "mc:40:9", "--blocks", "4", "--overlap", "0.1"])
    cfg = _config(args)
    assert (cfg.initial_guess, cfg.mc_samples, cfg.mc_seed) == ("mc", 40, 9)
    part = _partition(args, 100)
    assert part.k == 4
    args = ap.parse_args(["invert", "--in", "x", "--ordering", "red-black", "--overlap", "0.1"])
    with pytest.raises(ValueError):
        _partition(args, 100)
    args = ap.parse_args(["invert", "--in", "x", "--guess", "bogus"])
    with pytest.raises(ValueError):
        _config(args)


def test_cli_gen_and_error_exit(tmp_path, capsys):
    out = tmp_path / "c1.ibmi"
    assert main(["gen", "--config", "c1", "--out", str(out)]) == 0
    assert matio.read_header(out) == (512, 512)
    assert main(["invert", "--in", str(tmp_path / "missing.ibmi")]) == 1      # OSError -> exit 1
    assert "error:" in capsys.readouterr().err
