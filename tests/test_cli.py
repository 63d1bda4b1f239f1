"""CLI: usage/exit codes and text I/O on CPU; a JSON line per bench on the GPU."""
import json

import numpy as np
import pytest

from paper_1707_05141_b200 import cli


def test_no_arguments_is_usage_exit_1(capsys):
    assert cli.main([]) == 1
    assert "usage" in capsys.readouterr().err.lower()


def test_unknown_flag_is_usage_exit_1(capsys):
    assert cli.main(["bench", "svd", "--bogus", "1"]) == 1
    assert cli.main(["bench"]) == 1
    assert cli.main(["compress", "--n", "0"]) == 1
    assert cli.main(["compress", "--eps", "-1"]) == 1
    assert cli.main(["compress", "--svd", "qr"]) == 1


def test_matrix_text_roundtrip(tmp_path):
    a = np.random.default_rng(0).standard_normal((5, 3))
    p = tmp_path / "a.txt"
    cli.write_matrix_text(p, a)
    b = cli.read_matrix_text(p)
    assert b.flags.f_contiguous
    np.testing.assert_array_equal(a, b)
    (tmp_path / "bad.txt").write_text("2 2\n1 2 3\n")
    with pytest.raises(ValueError):
        cli.read_matrix_text(tmp_path / "bad.txt")


@pytest.mark.gpu
def test_bench_svd_json_line(capsys):
    assert cli.main(["bench", "svd", "--m", "32", "--n", "32", "--batch", "10", "--precision", "f64"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["command"] == "bench svd" and rec["config"]["ordering"] == "serial"
    assert rec["recon_rel_max"] <= 1e-13 and rec["orth_u_max"] <= 1e-13 and all(rec["converged"])


@pytest.mark.gpu
def test_bench_other_ops_and_strict(tmp_path):
    rep = tmp_path / "r.jsonl"
    for op in (["qr", "--m", "64", "--n", "32"], ["rsvd", "--m", "64", "--n", "64", "--k", "8"],
               ["block-svd", "--m", "64", "--n", "64", "--block-width", "16"]):
        assert cli.main(["bench", *op, "--batch", "4", "--report", str(rep)]) == 0
    lines = [json.loads(x) for x in rep.read_text().splitlines()]
    assert [x["command"] for x in lines] == ["bench qr", "bench rsvd", "bench block-svd"]
    assert lines[0]["recon_rel_max"] <= 1e-14
    # one sweep cannot converge: --strict turns that into exit 2
    assert cli.main(["bench", "svd", "--batch", "4", "--max-sweeps", "1", "--strict", "--report", str(rep)]) == 2
    p = tmp_path / "g.txt"
    assert cli.main(["gen", "--m", "6", "--n", "4", "--seed", "3", "--out", str(p)]) == 0
    assert cli.read_matrix_text(p).shape == (6, 4)


@pytest.mark.gpu
def test_compress_strict_reports_convergence(tmp_path):
    """compress carries the batched SVDs' converged flags: the JSON line counts the entries that
    did not converge and --strict exits 2 when there are any (SPEC exit-code convention)."""
    import json

    rep = tmp_path / "c.jsonl"
    rc = cli.main(["compress", "--n", "512", "--leaf-size", "32", "--cheb-order", "4", "--strict",
                   "--report", str(rep), "--error-vectors", "4"])
    line = json.loads(rep.read_text().splitlines()[-1])
    assert line["svd_calls"] > 0 and line["nonconverged_entries"] == 0
    assert rc == 0
