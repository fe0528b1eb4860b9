"""Text matrix files and the CLI on the GPU, mirroring the
reference's tests/test_traffic.py::TestMatrixFiles and tests/test_cli.py, and
checked byte-for-byte against the reference CLI's own outputs
(tests/golden/cli_golden.json, made by tests/golden/make_cli_golden.py)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2510_14050_b200 import AggregateReport, BenchResult, MatrixFileError, TrafficMatrix, read_matrix, write_matrix
from paper_2510_14050_b200.cli import cmd_analyze, cmd_bench, cmd_generate, load_matrix_dir, main
from paper_2510_14050_b200.traffic import read_matrix_device

pytestmark = pytest.mark.gpu

HAND = TrafficMatrix(0, 2, [0, 2, 3], [0, 1, 1], [2, 1, 3])
HAND_REPORT = AggregateReport(6, 3, 2, 2, 2, 2)
CLI_GOLDEN = json.loads((Path(__file__).parent / "golden" / "cli_golden.json").read_text())


def _random_matrix(rng, window_id=0):
    dim = int(rng.integers(1, 300))
    n = int(rng.integers(0, 2000))
    s = rng.integers(0, dim, n)
    d = rng.integers(0, dim, n)
    keys, counts = np.unique(s * dim + d, return_counts=True)
    rows, cols = keys // dim, keys % dim
    row_ptr = np.zeros(dim + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=dim), out=row_ptr[1:])
    return TrafficMatrix(window_id, dim, row_ptr, cols, counts)


def test_file_shape_and_round_trip(tmp_path):
    write_matrix(HAND, tmp_path / "m.txt")
    assert (tmp_path / "m.txt").read_text() == "2 3\n0 0 2\n0 1 1\n1 1 3\n"
    assert read_matrix(tmp_path / "m.txt") == HAND
    dim, coo = read_matrix_device(tmp_path / "m.txt")
    assert dim == 2 and coo.stats9() == (6, 3, 3, 2, 3, 2, 2, 4, 2)


def test_round_trip_random_corpus(tmp_path):
    rng = np.random.default_rng(99)
    for k in range(60):
        m = _random_matrix(rng, window_id=k)
        path = tmp_path / f"m{k}.txt"
        write_matrix(m, path)
        assert read_matrix(path, window_id=k) == m


def test_large_values_and_wide_rows(tmp_path):
    dim = 2**31
    rows = np.array([0, 5, 2**31 - 1], np.int64)
    cols = np.array([2**31 - 1, 7, 0], np.int64)
    vals = np.array([1, 2**32 - 1, 123456789], np.int64)
    text = "%d 3\n" % dim + "".join(f"{r} {c} {v}\n" for r, c, v in zip(rows, cols, vals))
    (tmp_path / "w.txt").write_text(text)
    d, coo = read_matrix_device(tmp_path / "w.txt")
    keys, counts = coo.download()
    assert d == dim and counts.tolist() == vals.tolist()
    assert (keys >> np.uint64(32)).astype(np.int64).tolist() == rows.tolist()


def test_nnz_mismatch_rejected(tmp_path):
    path = tmp_path / "bad.txt"
    path.write_text("3 5\n0 0 1\n0 1 1\n1 1 1\n2 2 1\n")
    with pytest.raises(MatrixFileError, match="claims 5 entries, file has 4"):
        read_matrix(path)


@pytest.mark.parametrize("content,match", [
    ("", "header"), ("3\n", "header"), ("a b\n", "header"), ("0 0\n", "dim must be"), ("2 -1\n", "nnz must be"),
    ("2 1\n0 0\n", "line 2"), ("2 1\n0 0 x\n", "line 2"), ("2 1\n0 5 1\n", "outside"),
    ("2 1\n0 0 0\n", "value must be >= 1"), ("2 2\n0 1 1\n0 0 1\n", "sorted"), ("2 2\n0 1 1\n0 1 2\n", "sorted"),
    ("2 1\n0 -1 1\n", "outside"), ("2 2\n0 0 1\n1 1 0\n", "line 3"),
])
def test_malformed_files_rejected(tmp_path, content, match):
    path = tmp_path / "bad.txt"
    path.write_text(content)
    with pytest.raises(MatrixFileError, match=match):
        read_matrix(path)
    with pytest.raises(MatrixFileError, match=match):
        read_matrix_device(path)


TEXT_GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "text_golden.json").read_text())["cases"]


@pytest.mark.parametrize("k", range(len(TEXT_GOLDEN)))
def test_text_parse_matches_reference(tmp_path, k):
    """Device tokenizer / validator vs the reference's read_matrix on the same bytes
    (tests/golden/text_golden.json, made by the reference itself): accepted variants
    (CRLF, lone CR, VT/FF/FS/GS/RS breaks, US, tabs, signs, underscores, leading zeros,
    non-ASCII whitespace and digits, no final newline) parse to the same matrix; every
    malformed file raises the same exception with the same message (file and line)."""
    import base64

    case = TEXT_GOLDEN[k]
    path = tmp_path / "m.txt"
    path.write_bytes(base64.b64decode(case["bytes"]))
    if case["ok"]:
        m = read_matrix(path)
        assert (m.dim, m.row_ptr.tolist(), m.col_idx.tolist(), m.values.tolist()) == (
            case["dim"], case["row_ptr"], case["col_idx"], case["values"])
        dim, coo = read_matrix_device(path)
        assert dim == case["dim"] and coo.nnz == len(case["values"])
        coo.close()
    else:
        with pytest.raises(MatrixFileError) as ei:
            read_matrix(path)
        assert type(ei.value).__name__ == case["error"]
        assert str(ei.value) == case["message"].replace("{path}", str(path))


@pytest.mark.parametrize("g", range(len(CLI_GOLDEN)))
def test_generate_matches_reference_bytes(tmp_path, g):
    gold = CLI_GOLDEN[g]
    c = gold["case"]
    out = tmp_path / "data"
    manifest = cmd_generate(n=c["n"], address_space=c["space"], seed=c["seed"], window_size=c["window"],
                            out_dir=out, invalid_fraction=c["invalid"])
    assert manifest == gold["manifest"]
    got = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(out.iterdir())}
    assert got == gold["sha256"]
    reports, totals, result = cmd_analyze(out)
    assert [r.to_dict() for r in reports] == gold["reports"]
    assert totals.to_dict() == gold["totals"]
    assert result.packet_count == c["n"] and result.analysis_time <= result.end_to_end_time
    matrices, reloaded = load_matrix_dir(out)
    assert reloaded == manifest and len(matrices) == manifest["window_count"]
    assert sum(int(m.values.sum()) for m in matrices) == gold["totals"]["valid_packets"]


def test_analyze_hand_fixture_and_outputs(tmp_path, capsys):
    d = tmp_path / "fixture"
    d.mkdir()
    write_matrix(HAND, d / "window_00000.txt")
    reports, totals, result = cmd_analyze(d, out=tmp_path / "r.json")
    assert reports == [HAND_REPORT] and totals == HAND_REPORT and result.packet_count == 6
    payload = json.loads((tmp_path / "r.json").read_text())
    assert payload["totals"] == HAND_REPORT.to_dict() and payload["bench"]["packet_count"] == 6
    out = capsys.readouterr().out
    assert "totals: valid_packets=6 unique_links=3" in out and "packet_rate=" in out
    base = cmd_analyze(d)[:2]
    assert cmd_analyze(d, resources=4, workers_per_resource=1, batch_count=10)[:2] == base
    assert cmd_analyze(d, inline=True)[:2] == base


def test_errors_and_exit_codes(tmp_path, capsys):
    d = tmp_path / "fixture"
    d.mkdir()
    (d / "window_00000.txt").write_text("2 9\n0 0 1\n")
    with pytest.raises(MatrixFileError, match="window_00000"):
        cmd_analyze(d)
    assert main(["analyze", "--in", str(d)]) == 2
    assert main(["analyze", "--in", str(tmp_path / "missing")]) == 2
    assert "error:" in capsys.readouterr().err
    with pytest.raises(ValueError):
        cmd_bench(d, [1], [1], repeats=0)


def test_bench_rows(tmp_path):
    d = tmp_path / "fixture"
    d.mkdir()
    write_matrix(HAND, d / "window_00000.txt")
    rows = cmd_bench(d, resource_list=[1, 2], batch_list=[1, 5], repeats=2, out=tmp_path / "b.jsonl")
    assert len(rows) == 4 and all(r["totals"] == HAND_REPORT.to_dict() for r in rows)
    lines = (tmp_path / "b.jsonl").read_text().splitlines()
    assert [json.loads(x)["resources"] for x in lines] == [1, 1, 2, 2]
    from paper_2510_14050_b200 import RunConfig

    r = BenchResult.from_times(1.0, 2.0, 10, RunConfig(1))
    assert r.packet_rate == 5.0 and r.to_dict()["config"]["resources"] == 1
