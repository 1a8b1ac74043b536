"""CLI front end: parsing and exit codes on CPU, a short run on the GPU."""
import json

import numpy as np
import pytest

from paper_2603_19959_b200.cli import (CSV_HEADER, EXIT_CONFIG, EXIT_NO_PEAKS, EXIT_OK,
                                       TABLE2_PRESETS, main,
                                       parse_config)


def test_defaults_and_presets():
    cfg, _ = parse_config([])
    assert (cfg.radius, cfg.n_x, cfg.degree_x, cfg.dt, cfg.dim, cfg.n_base) == (6.0, 64, 2, 0.1, 3, 4)
    cfg, _ = parse_config(["--table2", "q3-4-1"])
    assert (cfg.degree, cfg.n_base, cfg.levels) == (3, 4, 1)
    assert "q4-8-0" in TABLE2_PRESETS and "q4-8-1" not in TABLE2_PRESETS
    assert len(TABLE2_PRESETS) == 27


def test_config_errors_exit_2(capsys):
    assert main(["--table2", "q9-9-9"]) == EXIT_CONFIG
    assert main(["--not-a-flag"]) == EXIT_CONFIG
    assert main(["--Nb", "0"]) == EXIT_CONFIG
    capsys.readouterr()


@pytest.mark.gpu
def test_run_writes_outputs(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    csv, plot, summ = tmp_path / "o.csv", tmp_path / "p.py", tmp_path / "s.json"
    code = main(["--dv", "1", "--Nb", "16", "--p", "2", "--Nx", "16", "--steps", "60",
                 "--csv", str(csv), "--plot-script", str(plot), "--summary", str(summ)])
    out = json.loads(capsys.readouterr().out)
    assert code == EXIT_OK and out["n_peaks"] >= 2
    lines = csv.read_text().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 62
    data = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])
    assert abs(data[0, 1] - 0.02) < 1e-3
    assert json.loads(summ.read_text())["cells"] == 16
    assert "semilogy" in plot.read_text()


# The reference CLI suite's behaviours on the GPU run (pkg/tests/test_cli.py:55-141):
# %.17e CSV cells, per-step mass column with periodic bc, byte-identical reruns, the
# "---" sentinel with exit 4 when fewer than two peaks exist, exit 3 on an unwritable path.
SHORT = ["--dv", "1", "--Nb", "16", "--p", "2", "--Nx", "16", "--steps", "3"]


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_flags_parse_on_cpu():
    cfg, ns = parse_config(["--force-slow-path", "--workers", "3", "--dv", "1", "--bc",
                            "periodic", "--summary", "x.json"])
    assert cfg.force_slow and cfg.workers == 3 and cfg.dim == 1 and cfg.bc == "periodic"
    assert ns.summary == "x.json"


@pytest.mark.gpu
def test_csv_cells_are_17_digit_scientific(tmp_path, capsys):
    _gpu()
    csv = tmp_path / "c.csv"
    assert main(SHORT[:-1] + ["40", "--csv", str(csv), "--plot-script",
                              str(tmp_path / "p.py")]) in (EXIT_OK, EXIT_NO_PEAKS)
    capsys.readouterr()
    lines = csv.read_text().splitlines()
    assert float(lines[1].split(",")[0]) == 0.0
    for line in lines[1:3]:
        for tok in line.split(","):
            assert len(tok.split("e")[0].split(".")[1]) == 17


@pytest.mark.gpu
def test_periodic_mass_column_constant(tmp_path, capsys):
    _gpu()
    csv = tmp_path / "m.csv"
    assert main(SHORT[:-1] + ["60", "--bc", "periodic", "--csv", str(csv), "--plot-script",
                              str(tmp_path / "p.py")]) == EXIT_OK
    capsys.readouterr()
    m0 = np.genfromtxt(csv, delimiter=",", names=True)["m0"]
    assert np.abs(m0 - m0[0]).max() <= 1e-11 * abs(m0[0])


@pytest.mark.gpu
def test_rerun_writes_identical_bytes(tmp_path, capsys):
    _gpu()
    paths = [tmp_path / "r1.csv", tmp_path / "r2.csv"]
    for p in paths:
        assert main(SHORT + ["--csv", str(p), "--plot-script", str(tmp_path / "p.py")]) in (
            EXIT_OK, EXIT_NO_PEAKS)
    capsys.readouterr()
    assert paths[0].read_bytes() == paths[1].read_bytes()


@pytest.mark.gpu
def test_too_few_peaks_gives_sentinel_and_exit_4(tmp_path, capsys):
    _gpu()
    from paper_2603_19959_b200.cli import EXIT_NO_PEAKS as NOPK
    summ = tmp_path / "s.json"
    code = main(SHORT + ["--csv", str(tmp_path / "s.csv"), "--plot-script",
                         str(tmp_path / "p.py"), "--summary", str(summ)])
    capsys.readouterr()
    assert code == NOPK == 4
    d = json.loads(summ.read_text())
    assert d["gamma"] == "---" and d["rate_error_pct"] == "---"
    assert (tmp_path / "s.csv").exists()


@pytest.mark.gpu
def test_unwritable_output_exits_3(tmp_path, capsys):
    _gpu()
    code = main(SHORT + ["--csv", str(tmp_path / "missing" / "dir" / "x.csv"),
                         "--plot-script", str(tmp_path / "p.py")])
    capsys.readouterr()
    assert code == 3
