"""Summarise gpurun_out ncu artefacts into profiles/ (tracked).

usage: python tools/ncu_summary.py <tag> <launches.csv|-> [<prof.ncu-rep>] [--config cfg2]
Writes profiles/<tag>_launches.txt (per-kernel share of the step from the
gpu__time_duration launch list) and profiles/<tag>_ncu_full.txt (key metrics
per captured launch), and updates profiles/ncu_summary.json with the sweep
kernel's DRAM bytes per launch (read by bench.py as roofline.traffic).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "lts__t_bytes.sum",
        "smsp__inst_executed.sum"]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
              "GB": 1e9}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[d["Metric Unit"]]
                agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]) * scale)
    tot = sum(sum(v) for v in agg.values())
    lines = ["share   launches  mean_us  kernel  (ncu gpu__time_duration, cold-cache serialised)"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{100 * sum(v) / tot:5.1f}%  {len(v):6d}  {sum(v) / len(v):9.1f}  {k}")
    return "\n".join(lines)


def full(path):
    if path.endswith(".csv"):   # an `ncu -i ... --page raw --csv` dump made on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    val = float(v)
                except ValueError:
                    continue
                if "bytes" in k:
                    val *= UNIT_SCALE.get(units[i], 1)
                if k == "gpu__time_duration.sum":
                    val *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(units[i], 1.0)
                d[k] = val
        res.append(d)
    return res


def main():
    tag = sys.argv[1]
    cfg = "cfg2"
    if "--config" in sys.argv:
        cfg = sys.argv[sys.argv.index("--config") + 1]
    args = [a for a in sys.argv[2:] if not a.startswith("--") and a != cfg]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if args and args[0].endswith(".csv") and not args[0].endswith("_raw.csv"):
        txt = launches(args[0])
        open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w").write(txt + "\n")
        print(txt)
    rep = [a for a in args if a.endswith(".ncu-rep") or a.endswith("_raw.csv")]
    if rep:
        res = full(rep[0])
        lines = []
        for d in res:
            lines.append(d["kernel"])
            for k in KEYS:
                if k in d:
                    lines.append(f"    {k:60s} {d[k]:.6g}")
        open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.txt"), "w").write(
            "\n".join(lines) + "\n")
        print("\n".join(lines))
        summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
        summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
        for key, pat in (("sweep", "k_sweep_stream"), ("step_fused", "k_step_fused"),
                         ("xx", "k_xx_tiles")):
            hits = [d for d in res if pat in d["kernel"]]
            if not hits:
                continue
            s = hits[-1]
            summ.setdefault(cfg, {})[key] = {
                "kernel": s["kernel"], "tag": tag,
                "dram_bytes_per_launch": s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"],
                "duration_us_ncu": s["gpu__time_duration.sum"],
                "dram_throughput_pct": s.get(
                    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
        json.dump(summ, open(summ_path, "w"), indent=1)


if __name__ == "__main__":
    main()
