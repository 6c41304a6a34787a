"""I/O + CLI row against reference-generated fixtures (tests/golden/io,
make_golden_io.py): MatrixMarket read (values, canonicalisation, error messages and line numbers)
and write (byte-identical), VBR JSON round trip, CLI usage / runtime exit codes; the GPU tests
run the `block` and `bench` commands."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2202_05868_b200 import mtxio

IO = os.path.join(GOLDEN, "io")
EXPECT = json.load(open(os.path.join(IO, "expect.json")))
MTX = sorted(k for k in EXPECT if not k.startswith("cli_"))


@pytest.mark.parametrize("name", MTX)
def test_read_matrix_market_matches_reference(name):
    path = os.path.join(IO, f"{name}.mtx")
    exp = EXPECT[name]
    if "error" in exp:
        with pytest.raises(mtxio.MatrixMarketError) as ei:
            mtxio.read_matrix_market(path)
        assert str(ei.value).replace(path, "<path>") == exp["error"]
        assert ei.value.lineno == exp["lineno"]
        return
    A = mtxio.read_matrix_market(path)
    assert (A.n_rows, A.n_cols) == (exp["n_rows"], exp["n_cols"])
    assert A.row_ptr.tolist() == exp["row_ptr"] and A.col_idx.tolist() == exp["col_idx"]
    assert [repr(v) for v in A.values.tolist()] == exp["values"]


@pytest.mark.parametrize("name", [n for n in MTX if "error" not in EXPECT[n]])
def test_write_matrix_market_byte_identical(name, tmp_path):
    A = mtxio.read_matrix_market(os.path.join(IO, f"{name}.mtx"))
    out = tmp_path / "w.mtx"
    mtxio.write_matrix_market(out, A, comment="written by\nthe reference")
    assert out.read_bytes() == open(os.path.join(IO, f"{name}.written.mtx"), "rb").read()


def test_vbr_json_round_trip():
    from paper_2202_05868_b200.vbr import load_vbr, vbr_from_json, vbr_to_json

    V = load_vbr(os.path.join(IO, "cli_vbr.json"))
    doc = json.load(open(os.path.join(IO, "cli_vbr.json")))
    assert vbr_to_json(V) == doc
    W = vbr_from_json(vbr_to_json(V))
    assert np.array_equal(W.row_perm, V.row_perm) and W.stored_area == V.stored_area


def test_cli_usage_and_runtime_errors(tmp_path, capsys):
    from paper_2202_05868_b200 import cli

    with pytest.raises(SystemExit) as ei:
        cli.main(["block", "x.mtx", "--dw", "8", "--tau", "1.5"])
    assert ei.value.code == 2
    with pytest.raises(SystemExit) as ei:
        cli.main(["nope"])
    assert ei.value.code == 2
    assert cli.main(["block", str(tmp_path / "missing.mtx"), "--dw", "8", "--tau", "0.5"]) == 1
    assert "error:" in capsys.readouterr().err
    bad = os.path.join(IO, "bad_range.mtx")
    assert cli.main(["block", bad, "--dw", "8", "--tau", "0.5"]) == 1


@pytest.mark.gpu
def test_cli_block_matches_reference(tmp_path, capsys):
    from paper_2202_05868_b200 import cli

    out = tmp_path / "g.json"
    rc = cli.main(["block", os.path.join(IO, "cli_input.mtx"), "--dw", "8", "--tau", "0.3", "--out", str(out)])
    assert rc == EXPECT["cli_block"]["rc"] == 0
    assert capsys.readouterr().out == EXPECT["cli_block"]["stdout"]
    assert json.load(open(out)) == json.load(open(os.path.join(IO, "cli_grouping.json")))


@pytest.mark.gpu
def test_cli_bench_writes_rows(tmp_path, capsys):
    from paper_2202_05868_b200 import cli

    out = tmp_path / "bench.csv"
    rc = cli.main(["bench", os.path.join(IO, "cli_input.mtx"), "--dw", "8", "16", "--tau", "0.3", "-N", "64", "200",
                   "--runs", "2", "--out", str(out)])
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0].split(",") == cli.BENCH_COLUMNS + cli.GPU_COLUMNS
    rows = [dict(zip(lines[0].split(","), ln.split(","))) for ln in lines[1:]]
    assert len(rows) == 2 * 2 * 2 and {r["kernel"] for r in rows} == {"csr", "vbr"}
    assert all(float(r["median_s"]) > 0 for r in rows)
