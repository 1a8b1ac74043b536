"""Command-line front end over the GPU driver.

Same flags, `--table2` presets, CSV columns (`%.17e`), JSON summary and exit
codes as the reference front end (`sldg_vlasov/cli.py:13-57, 87-117, 165-193`),
so existing scripts keep working; the run itself goes through
`paper_2603_19959_b200.run` (device-resident Strang steps).
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from .driver import LANDAU_RATE_K05, SimConfig, run
from .sldg1d import ABSORBING, PERIODIC

EXIT_OK, EXIT_CONFIG, EXIT_RUNTIME, EXIT_NO_PEAKS = 0, 2, 3, 4
CSV_HEADER = "t,emax,m0,m1,m2,e_field,e_total"
# q<p>-<Nb>-<L>: uniform bases 3,4,5,6,8 and AMR (1 or 2 levels) on bases 3,4, p = 3..5
TABLE2_PRESETS = {}
for _p in (3, 4, 5):
    for _nb in (3, 4, 5, 6, 8):
        TABLE2_PRESETS[f"q{_p}-{_nb}-0"] = (_p, _nb, 0)
    for _nb in (3, 4):
        for _lv in (1, 2):
            TABLE2_PRESETS[f"q{_p}-{_nb}-{_lv}"] = (_p, _nb, _lv)

_FLAGS = [  # (flag, type, default, help, SimConfig field)
    ("--dv", int, 3, "velocity dimensions (1 or 3)", "dim"),
    ("--Nb", int, 4, "base velocity cells per dimension", "n_base"),
    ("--L", int, 0, "velocity AMR levels", "levels"),
    ("--R", float, 6.0, "velocity domain radius", "radius"),
    ("--p", int, 3, "velocity DG degree", "degree"),
    ("--Nx", int, 64, "spatial cells", "n_x"),
    ("--px", int, 2, "spatial DG degree", "degree_x"),
    ("--k", float, 0.5, "perturbation wave number", "wave_number"),
    ("--alpha", float, 0.01, "perturbation amplitude", "perturbation"),
    ("--dt", float, 0.1, "time step", "dt"),
    ("--steps", int, 200, "number of time steps", "n_steps"),
    ("--workers", int, 1, "accepted for compatibility (GPU run)", "workers"),
]


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="sldg-b200",
                                 description="SLDG Vlasov-Poisson benchmark on a B200.")
    for flag, typ, default, text, _ in _FLAGS:
        ap.add_argument(flag, type=typ, default=default, help=text)
    ap.add_argument("--bc", choices=[ABSORBING, PERIODIC], default=ABSORBING)
    ap.add_argument("--force-slow-path", action="store_true")
    ap.add_argument("--table2", metavar="ROW", help="preset q<p>-<Nb>-<L>, e.g. q5-4-0")
    ap.add_argument("--csv", default="run.csv")
    ap.add_argument("--plot-script", default="plot_emax.py")
    ap.add_argument("--summary", default=None)
    return ap


def parse_config(argv):
    ns = build_parser().parse_args(argv)
    if ns.table2 is not None:
        key = ns.table2.lower()
        if key not in TABLE2_PRESETS:
            raise ValueError(f"unknown preset {ns.table2!r}; try e.g. q5-4-0")
        ns.p, ns.Nb, ns.L = TABLE2_PRESETS[key]
    fields = {field: getattr(ns, flag.lstrip("-")) for flag, _, _, _, field in _FLAGS}
    cfg = SimConfig(**fields, bc=ns.bc, force_slow=ns.force_slow_path).validate()
    return cfg, ns


def write_csv(path, records):
    rows = [CSV_HEADER] + [",".join(f"{v:.17e}" for v in (r.t, r.e_max, r.m0, r.m1, r.m2,
                                                          r.e_field, r.e_total))
                           for r in records]
    with open(path, "w", newline="\n") as fh:
        fh.write("\n".join(rows) + "\n")


def summarize(result) -> dict:
    fit = result.fit
    return {
        "gamma": fit.rate if fit.ok else "---",
        "rate_error_pct": (abs((fit.rate - LANDAU_RATE_K05) / LANDAU_RATE_K05) * 100.0
                           if fit.ok else "---"),
        "n_peaks": fit.n_peaks, "mass_error": result.mass_error,
        "energy_drift": result.energy_drift, "cells": result.n_cells, "ips": result.n_ips,
        "wall_time_s": result.wall_time,
    }


def write_plot_script(path, csv_path, fit):
    png = str(path).rsplit(".", 1)[0] + ".png"
    gamma = None if fit.rate is None else fit.rate
    icpt = None if fit.intercept is None else fit.intercept
    lines = [
        "#!/usr/bin/env python3",
        "# E_max history (semilog) with the detected peaks and the envelope fit.",
        "import numpy as np",
        "import matplotlib.pyplot as plt",
        f"d = np.genfromtxt({str(csv_path)!r}, delimiter=',', names=True)",
        f"pt, pv = np.array({np.asarray(fit.peak_times).tolist()}), "
        f"np.array({np.asarray(fit.peak_values).tolist()})",
        "fig, ax = plt.subplots(figsize=(7, 4.5))",
        "ax.semilogy(d['t'], d['emax'], '-', lw=1.2, label='E_max')",
        "if pt.size:",
        "    ax.semilogy(pt, pv, 'kv', ms=7, label='peaks')",
        f"gamma, icpt = {gamma!r}, {icpt!r}",
        "if gamma is not None:",
        "    tt = np.linspace(pt[0], pt[-1], 50)",
        "    ax.semilogy(tt, np.exp(icpt + gamma * tt), 'k--', label=f'fit: gamma = {gamma:.4f}')",
        "ax.set_xlabel('t'); ax.set_ylabel('E_max'); ax.legend(); ax.grid(True, which='both', alpha=0.3)",
        f"fig.tight_layout(); fig.savefig({png!r}, dpi=150); print('wrote', {png!r})",
    ]
    with open(path, "w", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    try:
        cfg, ns = parse_config(argv)
    except SystemExit as exc:
        return EXIT_CONFIG if exc.code else EXIT_OK
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    try:
        result = run(cfg)
    except Exception as exc:  # noqa: BLE001 -- report and signal failure
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME
    try:
        write_csv(ns.csv, result.records)
        write_plot_script(ns.plot_script, ns.csv, result.fit)
        text = json.dumps(summarize(result), indent=2)
        print(text)
        if ns.summary:
            with open(ns.summary, "w", newline="\n") as fh:
                fh.write(text + "\n")
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME
    return EXIT_OK if result.fit.ok else EXIT_NO_PEAKS
