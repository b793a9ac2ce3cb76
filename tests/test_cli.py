"""CLI front end (mirrors the reference's cli.py tests, test_cli.py:8-153):
host-only commands run here; GPU commands are marked gpu."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2506_03686_b200 import TensorLayout
from paper_2506_03686_b200.cli import main, read_tensor, write_tensor


def test_vpt1_round_trip(tmp_path):
    lay = TensorLayout.from_shape((7, 32, 32, 3), 4)
    data = np.arange(lay.num_elements, dtype=np.uint32)
    p = tmp_path / "t.vpt"
    write_tensor(str(p), data, lay)
    lay2, payload = read_tensor(str(p))
    assert lay2 == lay and np.array_equal(payload.view(np.uint32), data)
    raw = p.read_bytes()
    assert raw[:4] == b"1TPV"                 # magic 0x56505431 little-endian


def test_plan_command(capsys):
    assert main(["plan", "--shape", "7,32,32,3", "--map", "0,2,3,1"]) == 0
    out = capsys.readouterr().out
    assert "kernel class" in out and "(0, 2, 3, 1)" in out


def test_gen_command(tmp_path, capsys):
    path = tmp_path / "k.cu"
    assert main(["gen", "--shape", "512,384", "--map", "1,0", "--out", str(path)]) == 0
    assert "vpg_tile_jit" in path.read_text()


def test_error_lines(tmp_path, capsys):
    assert main(["plan", "--map", "1,0"]) == 1
    assert "error missing-shape" in capsys.readouterr().err
    assert main(["plan", "--shape", "3,4", "--map", "0,0"]) == 1
    assert "error bad-map" in capsys.readouterr().err
    bad = tmp_path / "bad.vpt"
    bad.write_bytes(b"XXXX" * 4)
    assert main(["run", "--in", str(bad), "--map", "0"]) == 1
    assert "error bad-tensor-file" in capsys.readouterr().err


@pytest.mark.gpu
def test_run_against_oracle_file(cuda, tmp_path):
    """Paper shape (7,32,32,3) numpy map (0,2,3,1) via VPT1 files (test_cli.py:69-83)."""
    import oracle

    lay = TensorLayout.from_shape((7, 32, 32, 3), 4)
    data = np.random.default_rng(5).integers(0, 2**32 - 1, size=lay.num_elements, dtype=np.uint32)
    src, dst = tmp_path / "in.vpt", tmp_path / "out.vpt"
    write_tensor(str(src), data, lay)
    assert main(["run", "--in", str(src), "--map", "0,2,3,1", "--out", str(dst)]) == 0
    _, got = read_tensor(str(dst))
    dims, sigma = oracle.from_numpy_axes((7, 32, 32, 3), (0, 2, 3, 1))
    assert np.array_equal(got.view(np.uint32), oracle.naive_permute_c(data, dims, sigma))


@pytest.mark.gpu
def test_check_campaign(cuda, capsys):
    assert main(["check", "--cases", "200", "--seed", "2024"]) == 0
    assert "passed 200/200" in capsys.readouterr().out


@pytest.mark.gpu
def test_run_bounded_device_scratch(cuda, tmp_path):
    """`run --max-device-bytes` streams the tensor through a small device
    scratch; the output file matches the oracle."""
    import oracle

    shape, axes = (16, 64, 56, 56), (0, 2, 3, 1)
    x = np.random.default_rng(3).integers(0, 2**31, size=shape, dtype=np.uint32)
    src, dst = tmp_path / "x.vpt", tmp_path / "y.vpt"
    write_tensor(str(src), x.reshape(-1), TensorLayout.from_shape(shape, 4))
    assert main(["run", "--in", str(src), "--map", "0,2,3,1", "--out", str(dst),
                 "--max-device-bytes", str(4 << 20)]) == 0
    _, got = read_tensor(str(dst))
    dims, sigma = oracle.from_numpy_axes(shape, axes)
    assert np.array_equal(np.asarray(got).view(np.uint32).reshape(-1), oracle.naive_permute_c(x.reshape(-1), dims, sigma))
