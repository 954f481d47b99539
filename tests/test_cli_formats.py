"""Callers and data formats either side of the hot path,
CPU only: ATAM files bit-exact against files the reference wrote, the CLI's
argument rules / CSV schema / --dump-tree output against the reference, and
the distributed tree's retrieve-phase counters."""
import csv
import json
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2110_13042_b200 import cli, dist, read_matrix, write_matrix
from paper_2110_13042_b200.errors import ShapeMismatchError
from paper_2110_13042_b200.tasktree import build_tree_distributed, render_tree

GOLD = Path(__file__).parent / "golden"


def test_atam_reads_reference_files_and_roundtrips(tmp_path):
    rng = np.random.default_rng(5)              # the draws tools/make_golden_cli.py wrote
    f64 = rng.uniform(-1, 1, (7, 5))
    f32 = rng.standard_normal((3, 11)).astype(np.float32)
    for name, want in (("ref_f64.atam", f64), ("ref_f32.atam", f32)):
        got = read_matrix(GOLD / name)
        assert got.a.dtype == want.dtype and np.array_equal(got.a, want)
        out = tmp_path / name
        write_matrix(out, got)
        assert out.read_bytes() == (GOLD / name).read_bytes()     # byte-identical files


def test_atam_errors(tmp_path):
    bad = tmp_path / "bad.atam"
    bad.write_bytes(b"NOPE" + bytes(24))
    with pytest.raises(ValueError):
        read_matrix(bad)
    bad.write_bytes(b"ATAM" + struct.pack("<QQQ", 2, 2, 2) + bytes(8))
    with pytest.raises(ValueError):
        read_matrix(bad)
    with pytest.raises(ShapeMismatchError):
        write_matrix(tmp_path / "i.atam", np.ones((2, 2), dtype=np.float16))


def test_cli_csv_schema_matches_reference(tmp_path):
    g = json.loads((GOLD / "cli_csv.json").read_text())
    assert cli.CSV_HEADER == g["header"]
    r1 = cli.BenchRecord(mode="seq", m=1024, n=1024, procs=1, threshold=4096, reps=5,
                         median_s=0.123456789, eff_gflops=8.6975e3, max_abs_err=1.25e-13,
                         mult_count=362086400)
    r2 = cli.BenchRecord(mode="oracle", m=7, n=5, procs=1, threshold=32768, reps=1,
                         median_s=3.0e-05, eff_gflops=0.0058333)
    assert [[str(x) for x in r.csv_row()] for r in (r1, r2)] == [[str(x) for x in row] for row in g["rows"]]
    path = tmp_path / "out.csv"
    cli.write_csv(str(path), [r1])
    cli.write_csv(str(path), [r2])
    rows = list(csv.reader(open(path)))
    assert rows[0] == g["header"] and len(rows) == 3
    from paper_2110_13042_b200.measure import check_tolerance
    assert check_tolerance(np.full((7, 5), 0.5)) == pytest.approx(g["tolerance_f64_7x5"], rel=1e-15)
    assert check_tolerance(np.full((3, 11), 2.0, dtype=np.float32)) == \
        pytest.approx(g["tolerance_f32_3x11"], rel=1e-15)


def test_cli_argument_rules(monkeypatch):
    p = cli.build_parser()
    a = p.parse_args(["--mode", "shared"])
    cli.validate(a)
    assert a.procs == 1 and a.m == a.n == 1024 and a.threshold == 32768
    monkeypatch.setenv("ATA_THRESHOLD", "4096")
    a = p.parse_args(["--n", "100", "--m", "300"])
    cli.validate(a)
    assert (a.m, a.n, a.threshold) == (300, 100, 4096)
    with pytest.raises(SystemExit):
        cli.validate(p.parse_args(["--mode", "seq", "--procs", "2"]))
    with pytest.raises(SystemExit):
        cli.validate(p.parse_args(["--mode", "seq", "--comm-csv", "x.csv"]))
    a = p.parse_args(["--mode", "auto"])
    cli.validate(a)
    assert a.threshold == "auto"


def test_cli_dump_tree_matches_reference(capsys):
    trees = json.loads((GOLD / "trees.json").read_text())["cases"]
    for mode, flag in (("distributed", "dist"), ("shared", "shared")):
        case = next(c for c in trees if c["mode"] == mode and c["p"] == 8 and c["m"] == 65536)
        assert cli.main(["--mode", flag, "--procs", "8", "--m", "65536", "--n", "32768", "--dump-tree"]) == 0
        assert capsys.readouterr().out.rstrip("\n") == case["render"]


def test_tree_comm_stats_and_csv(tmp_path):
    t = build_tree_distributed(8, 65536, 32768)
    st = dist.tree_comm_stats(t)
    assert st["sent_messages"][0] == 0 and sum(st["sent_messages"]) == 7
    assert sum(st["sent_words"]) == sum(st["recv_words"])
    tri = 16384 * 16385 // 2
    # p1 sends C11's partial to p0; p6 sends its C21 tile to p4; p4 sends C21 to p0
    assert st["sent_words"][1] == tri and st["sent_words"][6] == 8192 * 16384
    assert st["sent_words"][4] == 16384 * 16384
    path = tmp_path / "comm.csv"
    dist.write_comm_csv(path, st, 8)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["process", "sent_messages", "sent_words", "recv_messages", "recv_words"]
    assert rows[-1][0] == "critical_path" and len(rows) == 10
    assert "bunch" in render_tree(t)
