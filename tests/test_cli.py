"""CLI harness (paper_2403_06348_b200/cli.py): report schema, exit codes and
config echo of pkg/src/alto/cli.py, the cases of pkg/tests/test_cli.py run
against the GPU path, plus CP-ALS / CP-APR results checked against the
oracle drivers. Error paths that fail before touching the device run on CPU."""

import io
import json

import numpy as np
import pytest

from conftest import EXAMPLE_COORDS, EXAMPLE_DIMS, EXAMPLE_VALUES, random_sparse

from paper_2403_06348_b200 import cli

EXAMPLE_TNS = "".join(" ".join(str(c + 1) for c in row) + f" {v}\n"
                      for row, v in zip(EXAMPLE_COORDS, EXAMPLE_VALUES))


def run(capsys, *argv):
    code = cli.main([str(a) for a in argv])
    out = capsys.readouterr()
    return code, (json.loads(out.out) if out.out.strip() else None), out.err


@pytest.fixture()
def example_file(tmp_path):
    p = tmp_path / "example.tns"
    p.write_text(EXAMPLE_TNS)
    return str(p)


def _write_tns(path, coords, values):
    with open(path, "w") as f:
        for row, v in zip(coords, values):
            f.write(" ".join(str(int(c) + 1) for c in row) + f" {float(v)!r}\n")


# ---------------------------------------------------------------- CPU


def test_usage_error(capsys):
    code, payload, _ = run(capsys, "frobnicate")
    assert code == cli.EXIT_USAGE and payload["error"]["type"] == "usage"
    code, payload, _ = run(capsys, "bench", "mttkrp")  # missing input
    assert code == cli.EXIT_USAGE


def test_missing_file_is_input_error(capsys):
    code, payload, err = run(capsys, "stats", "/no/such/file.tns")
    assert code == cli.EXIT_INPUT
    assert payload["error"]["type"] == "FileNotFoundError" and err.startswith("error:")


@pytest.mark.gpu  # the parse stages into pinned host memory
def test_parse_error_leaves_no_output(capsys, tmp_path):
    bad = tmp_path / "bad.tns"
    bad.write_text("1 1 not_a_number\n")
    out = tmp_path / "out.alto"
    code, payload, _ = run(capsys, "convert", bad, out)
    assert code == cli.EXIT_INPUT and payload["error"]["type"] == "ParseError"
    assert "bad value" in payload["error"]["message"]
    assert not out.exists() and list(tmp_path.iterdir()) == [bad]


def test_parse_dims():
    assert cli.parse_dims("4,8,2") == (4, 8, 2)
    assert cli.parse_dims("4x8x2") == (4, 8, 2)
    assert cli.parse_dims(None) is None
    with pytest.raises(ValueError):
        cli.parse_dims("4,a")
    with pytest.raises(ValueError):
        cli.parse_dims(",")


def test_default_threads_env(monkeypatch):
    monkeypatch.setenv("ALTO_THREADS", "3")
    assert cli.default_threads() == 3
    monkeypatch.setenv("ALTO_THREADS", "junk")
    assert cli.default_threads() >= 1


def test_parser_defaults():
    a = cli.build_parser().parse_args(["cp-apr", "x.tns"])
    assert (a.rank, a.max_outer, a.max_inner, a.mem, a.eps) == (16, 200, 10, "auto", 1e-10)
    a = cli.build_parser().parse_args(["bench", "mttkrp", "x.tns"])
    assert (a.rank, a.mode, a.iters, a.strategy, a.temp_budget_bytes) == (16, "all", 3, "auto", 1 << 30)


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_stats_worked_example(capsys, example_file):
    code, rep, _ = run(capsys, "stats", example_file, "--dims", "4,8,2", "--word-bits", "8",
                       "--partitions", "2")
    assert code == 0
    res = rep["result"]
    assert res["compression_ratio"] == 3.0
    segs = res["partitions"]["segments"]
    assert [(s["pos_first"], s["pos_last"]) for s in segs] == [(2, 20), (25, 51)]
    assert segs[0]["intervals"] == [[0, 3], [0, 3], [0, 1]]
    assert segs[1]["intervals"] == [[1, 3], [2, 6], [0, 1]]
    assert rep["tensor"] == {"dims": list(EXAMPLE_DIMS), "nnz": 6}
    assert set(rep) == {"command", "input", "version", "config", "timing_s", "tensor", "result"}


@pytest.mark.gpu
def test_convert_roundtrip(capsys, example_file, tmp_path):
    import paper_2403_06348_b200 as alto

    binpath, textpath = tmp_path / "t.alto", tmp_path / "back.tns"
    code, rep, _ = run(capsys, "convert", example_file, binpath, "--dims", "4,8,2")
    assert code == 0
    assert rep["result"]["format"] == "alto"
    assert (rep["result"]["index_bits"], rep["result"]["position_bits"]) == (6, 64)
    assert {"parse_s", "linearize_s", "sort_s", "write_s"} <= set(rep["timing_s"])
    code, rep, _ = run(capsys, "convert", binpath, textpath)
    assert code == 0 and rep["result"]["format"] == "tns" and "read_s" in rep["timing_s"]
    back = alto.parse_frostt(str(textpath), dims=EXAMPLE_DIMS)
    orig = alto.parse_frostt(io.StringIO(EXAMPLE_TNS), dims=EXAMPLE_DIMS)
    assert back == orig
    t = alto.read_alto(str(binpath))
    assert t.shape.dims == EXAMPLE_DIMS and t.nnz == 6
    # --dims is for text input only
    code, payload, _ = run(capsys, "stats", binpath, "--dims", "4,8,2")
    assert code == cli.EXIT_INPUT and "--dims" in payload["error"]["message"]


@pytest.mark.gpu
@pytest.mark.parametrize("exact", [False, True])
def test_bench_report(capsys, example_file, exact):
    extra = ["--exact"] if exact else []
    code, rep, err = run(capsys, "bench", "mttkrp", example_file, "--dims", "4,8,2", "--rank", "2",
                         "--iters", "2", "--threads", "2", "--mode", "all", *extra)
    assert code == 0
    per = rep["result"]["per_mode"]
    assert [e["mode"] for e in per] == [0, 1, 2]
    for e in per:
        assert e["median_s"] >= 0 and len(e["times_s"]) == 2 and len(e["device_times_s"]) == 2
        assert e["flops_per_nonzero"] == 2 * 2 * 2 + 2
        assert e["strategy"]["strategy"] in ("sequential", "recursive", "output")
        assert e["gpu"]["kernel"] and e["gpu"]["mode"] == e["mode"]
    assert rep["config"]["threads"] == 2 and rep["config"]["partitions"] == 2
    assert rep["config"]["exact"] is exact
    assert err.startswith("bench mttkrp:")
    code, rep, _ = run(capsys, "bench", "mttkrp", example_file, "--dims", "4,8,2", "--mode", "1",
                       "--iters", "1")
    assert code == 0 and [e["mode"] for e in rep["result"]["per_mode"]] == [1]


@pytest.mark.gpu
def test_cp_als_model_file_matches_oracle(capsys, tmp_path):
    from oracle import alto_oracle as orc

    rng = np.random.default_rng(11)
    dims = (9, 7, 6)
    coords, vals = random_sparse(rng, dims, 120)
    path = tmp_path / "x.tns"
    _write_tns(path, coords, vals)
    out = tmp_path / "model.json"
    code, rep, _ = run(capsys, "cp-als", path, "--dims", "9,7,6", "--rank", "3", "--max-iters", "6",
                       "--tol", "1e-300", "--seed", "1", "--out", out)
    assert code == 0
    model = json.loads(out.read_text())
    assert model["shape"] == list(dims) and model["rank"] == 3
    assert len(model["lambda"]) == 3 and [len(f) for f in model["factors"]] == list(dims)
    assert model["trace"]["iterations"] == rep["result"]["iterations"] == 6
    assert "wall_time_s" in model["trace"] and rep["result"]["out"] == str(out)
    _keys, svals, scoords = orc.from_coo(dims, coords, vals)
    w, f, fits = orc.cp_als(dims, scoords, svals, 3, 6, seed=1)
    np.testing.assert_allclose(model["trace"]["fit"], fits, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(rep["result"]["lambda"], w, rtol=1e-9)


@pytest.mark.gpu
def test_cp_apr_model_file_matches_oracle(capsys, tmp_path):
    from oracle import alto_oracle as orc

    rng = np.random.default_rng(50)
    dims = (5, 4, 3)
    coords, vals = random_sparse(rng, dims, 25, kind="counts")
    path = tmp_path / "c.tns"
    _write_tns(path, coords, vals)
    out = tmp_path / "model.json"
    code, rep, _ = run(capsys, "cp-apr", path, "--dims", "5,4,3", "--rank", "2", "--seed", "2",
                       "--max-outer", "20", "--out", out)
    assert code == 0
    model = json.loads(out.read_text())
    assert model["trace"]["memory_mode"] == "otf" and rep["config"]["memory_mode_used"] == "otf"
    keys, svals, scoords = orc.from_coo(dims, coords, vals)
    w, f, kkt, inner, ll = orc.cp_apr(dims, scoords, svals, 2, 20, seed=2)
    assert model["trace"]["inner_iters"] == list(inner)
    np.testing.assert_allclose(model["trace"]["kkt"], kkt, rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(model["trace"]["loglik"], ll, rtol=1e-9)
    assert rep["result"]["final_kkt"] == max(model["trace"]["kkt"][-1])


@pytest.mark.gpu
def test_inline_model_and_config_echo(capsys, example_file, monkeypatch):
    code, rep, _ = run(capsys, "cp-als", example_file, "--dims", "4,8,2", "--rank", "1", "--max-iters", "3")
    assert code == 0 and "model" in rep["result"] and "out" not in rep["result"]
    code, rep, _ = run(capsys, "cp-als", example_file, "--dims", "4,8,2", "--rank", "2", "--max-iters", "2",
                       "--threads", "2")
    cfg = rep["config"]
    assert (cfg["rank"], cfg["threads"], cfg["partitions"], cfg["strategy"]) == (2, 2, 2, "auto")
    monkeypatch.setenv("ALTO_THREADS", "3")
    code, rep, _ = run(capsys, "cp-als", example_file, "--dims", "4,8,2", "--rank", "1", "--max-iters", "1")
    assert code == 0 and rep["config"]["threads"] == 3


@pytest.mark.gpu
def test_cp_apr_negative_input_is_input_error(capsys, tmp_path):
    p = tmp_path / "neg.tns"
    p.write_text("1 1 1 1.0\n2 2 2 -3.0\n")
    code, payload, _ = run(capsys, "cp-apr", p, "--rank", "1")
    assert code == cli.EXIT_INPUT and "negative" in payload["error"]["message"]


@pytest.mark.gpu
def test_module_entry_point(tmp_path, example_file):
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "-m", "paper_2403_06348_b200", "stats", example_file,
                        "--dims", "4,8,2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["result"]["dims"] == list(EXAMPLE_DIMS)
