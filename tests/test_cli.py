"""CLI and file formats (cli.py:131-209, sparse.py:152-173, chains.py:370-447).

CPU: argument parsing, Matrix Market round trips, chain import and the Petri
JSON reader.  GPU: `solve` / `table` / `gen` end to end, twice, byte-identical
files, and the solve agreeing with the reference's golden output.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
from scipy import sparse as sp

from paper_1402_4005_b200 import cli
from paper_1402_4005_b200.chains import import_chain, petri_spec_from_json, tandem_queue
from paper_1402_4005_b200.sparse import load_matrix_market, load_vector, save_matrix_market, save_vector


def test_parser_mirrors_reference_options():
    p = cli.build_parser()
    a = p.parse_args(["solve", "--family", "tandem", "--n", "1024", "--rtol", "1e-8", "--cycles", "2"])
    assert (a.family, a.n, a.rtol, a.cycles, a.max_iters, a.restart) == ("tandem", 1024, 1e-8, 2, 1000, 50)
    a = p.parse_args(["table", "--family", "planar", "--sizes", "1024,2048"])
    assert a.cap == 1000 and a.seed == 1
    with pytest.raises(SystemExit):
        p.parse_args(["solve", "--cycles", "3"])


def test_matrix_market_round_trip(tmp_path):
    prob = tandem_queue(9)
    save_matrix_market(tmp_path / "B.mtx", prob.B)
    B = load_matrix_market(tmp_path / "B.mtx")
    assert (B != prob.B).nnz == 0
    x = np.random.default_rng(1).standard_normal(prob.n)
    save_vector(tmp_path / "x.mtx", x)
    assert np.array_equal(load_vector(tmp_path / "x.mtx"), x)  # 17 digits: exact round trip


def test_import_chain_detects_A_and_B(tmp_path):
    prob = tandem_queue(7)
    save_matrix_market(tmp_path / "A.mtx", prob.A)
    save_matrix_market(tmp_path / "B.mtx", prob.B)
    for f in ("A.mtx", "B.mtx"):
        q = import_chain(tmp_path / f)
        assert q.family == "imported" and abs(q.B - prob.B).max() < 1e-15
    save_matrix_market(tmp_path / "bad.mtx", sp.csr_array(np.eye(3) * 0.5))
    with pytest.raises(ValueError, match="neither column-stochastic"):
        import_chain(tmp_path / "bad.mtx")


def test_petri_spec_json():
    doc = {"places": 2, "initial_marking": [1, 0],
           "transitions": [{"inputs": {"0": 1}, "outputs": {"1": 1}, "weight": 2.0},
                           {"inputs": {"1": 1}, "outputs": {"0": 1}}]}
    places, trans, marking = petri_spec_from_json(json.dumps(doc))
    assert places == 2 and marking == (1, 0) and trans[0][2] == 2.0 and trans[1][2] == 1.0


def test_missing_import_is_io_error(tmp_path):
    assert cli.main(["solve", "--import", str(tmp_path / "none.mtx"), "--out", str(tmp_path)]) == cli.IO_ERROR


@pytest.mark.gpu
def test_solve_outputs_deterministic_and_match_reference(tmp_path, golden):
    g = golden("pipe_bd257_normal")  # reference run: birth-death 257, seed 1, rtol 1e-7, normal init
    outs = []
    for rep in range(2):
        d = tmp_path / f"run{rep}"
        rc = cli.main(["solve", "--family", "birth-death", "--n", "257", "--seed", "1", "--out", str(d)])
        assert rc == 0
        outs.append({f: (d / f).read_bytes() for f in ("report.json", "x.mtx", "residuals.csv", "manifest.json")})
    assert outs[0] == outs[1]
    doc = json.loads(outs[0]["report.json"])
    assert doc["converged"] and doc["n"] == 257 and doc["family"] == "birth-death"
    assert abs(doc["iterations"] - int(g["iterations"])) <= 1
    x = load_vector(tmp_path / "run0" / "x.mtx")
    assert np.abs(x - g["x"]).sum() <= 1e-8
    assert "seconds" not in outs[0]["report.json"].decode()  # no timings in files


@pytest.mark.gpu
def test_table_and_gen(tmp_path):
    rc = cli.main(["table", "--family", "uniform2d", "--sizes", "289,1089", "--out", str(tmp_path)])
    assert rc == 0
    lines = (tmp_path / "table.csv").read_text().strip().splitlines()
    assert lines[0].startswith("family,row,n") and len(lines) == 1 + 3 * 2
    assert all(",True," in ln for ln in lines[1:])
    rc = cli.main(["gen", "--family", "tandem", "--n", "64", "--out", str(tmp_path / "gen")])
    assert rc == 0 and (tmp_path / "gen" / "B.mtx").exists()
