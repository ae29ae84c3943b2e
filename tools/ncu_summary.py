"""Summarise ncu captures (run here, on the CPU box) into profiles/.

  python tools/ncu_summary.py <tag> gpurun_out/prof_G.ncu-rep [...]   -> profiles/<tag>_ncu.json + .md
  python tools/ncu_summary.py <tag> --launches gpurun_out/launches_G.csv
  python tools/ncu_summary.py <tag> --traffic best.json gpurun_out/prof_*.ncu-rep
      -> also merges DRAM bytes per launch of every captured kernel into
         profiles/ncu_traffic.json {"kernels": {name: {...}}} (bench.py reads it
         for roofline.traffic of the kernel it reports, and only that kernel)

For each --set full report: duration, DRAM bytes read/written (per launch),
DRAM throughput %, tensor-pipe %, warps active %, registers, grid/block, and
the top stall reasons of the source page when present.  For a launch list
(--metrics gpu__time_duration.sum): per-kernel-name counts and time shares.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "launch__cluster_dim_x": "cluster",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3}


def raw(report: str) -> list:
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")] if "Kernel Name" in head else "?"}
        for m, k in METRICS.items():
            if m not in head:
                continue
            i = head.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if k == "duration":
                v *= SCALE.get(u, 1.0)  # -> microseconds
            elif k in ("dram_read", "dram_write", "l2_bytes"):
                v *= SCALE.get(u, 1.0)  # -> bytes
            d[k] = v
        res.append(d)
    return res


def launches(path: str) -> dict:
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(lines))
    head = rows[0]
    ki, mi, vi, ui = (head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value"),
                      head.index("Metric Unit"))
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        name = "sgm_cand_*" if name.startswith("sgm_cand_") else name
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        per[name][0] += 1
        per[name][1] += v
    tot = sum(v[1] for v in per.values()) or 1.0
    return {k: {"launches": n, "time_us": t, "share": t / tot} for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1])}


def main(argv):
    tag = argv[0]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if argv[1] == "--traffic":
        best = json.load(open(argv[2]))
        res = {os.path.basename(p): raw(p) for p in argv[3:]}
        path = os.path.join(ROOT, "profiles", f"{tag}_ncu.json")
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        try:
            traffic = json.load(open(tpath))
        except Exception:
            traffic = {}
        kern = traffic.get("kernels", {}) if isinstance(traffic.get("kernels"), dict) else {}
        by_kernel = {b["kernel"]: w for w, b in best.items() if "kernel" in b}
        for w, b in best.items():
            for ru in b.get("runners_up", []):
                by_kernel.setdefault(ru["kernel"], w)
        for rep, rows in res.items():
            for r in rows:
                w = by_kernel.get(r["kernel"])
                kern[r["kernel"]] = {"workload": w, "dram_bytes": r.get("dram_read", 0) + r.get("dram_write", 0),
                                     "dram_read": r.get("dram_read"), "dram_write": r.get("dram_write"),
                                     "duration_us_ncu": r.get("duration"), "dram_pct": r.get("dram_pct"),
                                     "algorithmic_bytes": best[w]["algorithmic_bytes"] if w else None,
                                     "source": f"profiles/{tag}_ncu.json ({rep}, ncu --set full)"}
        with open(tpath, "w") as fh:
            json.dump({"what": "DRAM bytes (read + write) per launch of captured kernels, keyed by kernel name",
                       "kernels": kern}, fh, indent=1)
    elif argv[1] == "--launches":
        res = {os.path.basename(p): launches(p) for p in argv[2:]}
        path = os.path.join(ROOT, "profiles", f"{tag}_launches.json")
    else:
        res = {os.path.basename(p): raw(p) for p in argv[1:]}
        path = os.path.join(ROOT, "profiles", f"{tag}_ncu.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    main(sys.argv[1:])
