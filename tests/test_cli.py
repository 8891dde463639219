"""CLI / harness (reference pkg/tests/test_cli.py strategy) on the GPU package."""

import numpy as np
import pytest

from paper_1908_11807_b200 import datasets
from paper_1908_11807_b200.cli import main
from paper_1908_11807_b200.harness import CSV_HEADER, SCALE_CSV_HEADER, BenchConfig


# ----------------------------------------------------------------- CPU: host logic


def test_generate_writes_clouds(tmp_path, capsys):
    out = tmp_path / "c.pcl3"
    assert main(["generate", "--m", "1000", "--source", "sphere:hollow", str(out)]) == 0
    pts = datasets.load_cloud(out)
    assert pts.shape == (1000, 3)
    a, b = tmp_path / "a", tmp_path / "b"
    for p in (a, b):
        assert main(["generate", "--m", "500", "--seed", "4", str(p)]) == 0
    assert a.read_bytes() == b.read_bytes()
    csv = tmp_path / "c.csv"
    assert main(["generate", "--m", "10", str(csv)]) == 0
    assert csv.read_text().count("\n") == 10
    assert main(["generate", "--m", "10", str(tmp_path / "no" / "dir" / "x")]) == 2


@pytest.mark.parametrize("argv,needle", [
    (["bench", "--alloc", "1p"], "buffer-size"),
    (["bench", "--buffer-size", "4"], "only valid"),
    (["bench", "--kind", "knn", "--alloc", "2p"], "does not apply"),
    (["scale", "--threads", "1,x"], "comma-separated"),
    (["bench", "--m", "0"], "must be >= 1"),
])
def test_usage_errors_exit_1(argv, needle, capsys):
    assert main(argv) == 1
    assert needle in capsys.readouterr().err


def test_bad_subcommand_usage_error():
    with pytest.raises(SystemExit) as exc:
        main(["frobnicate"])
    assert exc.value.code == 1


def test_config_validation():
    BenchConfig(kind="spatial", alloc="1p", buffer_size=4).validate()
    with pytest.raises(ValueError):
        BenchConfig(source="cube:solid").validate()
    assert BenchConfig(k=10).effective_radius == datasets.default_radius(10)
    assert BenchConfig(kind="knn").effective_alloc == "-"


# ----------------------------------------------------------------- GPU: runs


@pytest.mark.gpu
def test_bench_csv_schema_and_kinds(capsys):
    assert main(["bench", "--m", "500", "--reps", "1", "--target", "cube:filled"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == CSV_HEADER
    row = lines[1].split(",")
    assert len(row) == len(CSV_HEADER.split(",")) and row[:4] == ["500", "500", "spatial", "2p"]
    assert main(["bench", "--m", "400", "--reps", "1", "--kind", "knn", "--sort-queries", "off"]) == 0
    row = capsys.readouterr().out.strip().splitlines()[1].split(",")
    assert row[2] == "knn" and row[3] == "-" and row[4] == "off" and float(row[11]) == 10.0
    assert main(["bench", "--m", "300", "--reps", "1", "--alloc", "1p", "--buffer-size", "2",
                 "--format", "pretty"]) == 0
    assert "queries/s" in capsys.readouterr().out


@pytest.mark.gpu
def test_scale_rows(capsys):
    assert main(["scale", "--m", "300", "--reps", "1", "--threads", "1,2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == SCALE_CSV_HEADER and len(lines) == 3
    r1, r2 = lines[1].split(","), lines[2].split(",")
    assert r1[-2:] == ["1.00", "1.00"] and r1[10:13] == r2[10:13]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["spatial", "knn"])
def test_verify_clean_and_corrupted(kind, capsys):
    assert main(["verify", "--m", "2000", "--kind", kind]) == 0
    assert "0 mismatched" in capsys.readouterr().out
    assert main(["verify", "--m", "2000", "--kind", kind, "--source", "cube:hollow",
                 "--target", "sphere:hollow"]) == 0
    capsys.readouterr()
    assert main(["verify", "--m", "2000", "--kind", kind, "--corrupt-tree"]) == 3
    assert main(["verify", "--m", "200000"]) == 1
