"""CLI front end: parsing and exit codes on CPU, a short run on the GPU."""
import json

import numpy as np
import pytest

from paper_2603_19959_b200.cli import (CSV_HEADER, EXIT_CONFIG, EXIT_OK, TABLE2_PRESETS, main,
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
