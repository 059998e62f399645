"""The b200 CLI (paper_2103_08825_b200/cli.py), modelled on the reference's
CLI tests: argument errors exit 2 with ``error:`` (cli.py:167-170), verify
exits 0/1 on the 1e-13-per-step bar (cli.py:120-127)."""

import pytest

from paper_2103_08825_b200.cli import main, parse_cli


@pytest.mark.parametrize("argv,match", [
    (["run", "--stencil", "1d3p", "--size", "0", "--method", "b200"], "positive"),
    (["run", "--stencil", "1d3p", "--size", "64", "--method", "b200", "--steps", "0"], "steps"),
    (["run", "--stencil", "2d9p", "--size", "64", "--method", "b200", "--block", "16", "--tile-height", "4"], "device"),
    (["run", "--stencil", "1d3p", "--size", "64", "--method", "b200", "--weights", "c5"], "d=3"),
    (["run", "--stencil", "1d3p", "--size", "64", "--method", "b200", "--weights", "1,2"], "needs 3 weights"),
    (["run", "--stencil", "1d3p", "--size", "64x9", "--method", "b200"], "needs 1 extents"),
    (["verify", "--stencil", "1d3p", "--size", "64", "--method", "b200", "--vl", "6"], "vl"),
])
def test_errors_exit_2(argv, match, capsys):
    assert main(argv) == 2
    err = capsys.readouterr().err
    assert err.startswith("error:") and match in err


def test_parse_broadcast_size_and_weights():
    a = parse_cli(["run", "--stencil", "3d27p", "--size", "16", "--method", "b200_dlt", "--weights", "c5",
                   "--jam-k", "2"])
    assert a.cfg.dims == (16, 16, 16) and a.cfg.jam_k == 2 and a.cfg.method == "b200_dlt"
    assert a.cfg.spec().name == "c5_3d27p"
    b = parse_cli(["run", "--stencil", "1d3p", "--size", "64", "--method", "b200", "--weights", "0.25,0.5,0.25"])
    assert [b.cfg.spec().weights[o] for o in b.cfg.spec().offsets] == [0.25, 0.5, 0.25]


def test_plan_prints_roofline(capsys):
    assert main(["plan", "--stencil", "3d7p", "--size", "512", "--weights", "c4"]) == 0
    out = capsys.readouterr().out
    assert "F=13" in out and "k= 2" in out and "device plan" in out


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["b200", "b200_transpose", "b200_dlt"])
def test_verify_passes_on_device(method, capsys):
    pytest.importorskip("stencilbench", reason="verify uses the reference oracle")
    assert main(["verify", "--stencil", "2d9p", "--size", "24x40", "--steps", "6", "--method", method]) == 0
    assert capsys.readouterr().out.startswith("PASS")


@pytest.mark.gpu
def test_run_fma_custom_weights_csv(tmp_path, capsys):
    pytest.importorskip("stencilbench", reason="--verify uses the reference oracle")
    csv = tmp_path / "r.csv"
    assert main(["run", "--stencil", "3d27p", "--size", "12x16x40", "--steps", "4", "--method", "b200",
                 "--weights", "c5", "--arith", "fma", "--jam-k", "2", "--verify", "--csv", str(csv)]) == 0
    out = capsys.readouterr().out
    assert "max rel err vs oracle" in out
    lines = csv.read_text().splitlines()
    assert lines[0].startswith("stencil,method") and lines[1].startswith("3d27p,b200,4,2,12x16x40,4,")
