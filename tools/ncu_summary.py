#!/usr/bin/env python
"""Summarize ncu evidence into profiles/<tag>_ncu_summary.json (+ a text table).

  python tools/ncu_summary.py --tag r1 --launches gpurun_out/launches.csv --full gpurun_out/prof_r1.ncu-rep

* launches: `ncu --metrics gpu__time_duration.sum --clock-control none --csv` of a bench run
  (cold-cache, serialised launches: per-kernel SHARE of the step is what matters)
* full: `ncu --set full` capture of the hot kernels -> per-launch DRAM bytes, duration,
  throughput, registers, occupancy (bench.py reads dram_bytes_per_launch as roofline.traffic)
"""
import argparse
import collections
import csv
import io
import json
import pathlib
import re
import subprocess

ROOT = pathlib.Path(__file__).resolve().parents[1]


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[\d, ]+>)?", name)
    return (m.group(1) + (m.group(2) or "").replace(" ", "")) if m else name[:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg[short(r[ki])].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    total = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / total}
            for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))}


def full(path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(h)}

    def val(r, name, to_bytes=False):
        if name not in col:
            return None
        s = r[col[name]].replace(",", "")
        try:
            v = float(s)
        except ValueError:
            return None
        if to_bytes:
            u = units[col[name]]
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        return v

    ks = collections.defaultdict(list)
    for r in rows[2:]:
        name = short(r[col["Kernel Name"]])
        dur_ms = val(r, "gpu__time_duration.sum")
        if units[col["gpu__time_duration.sum"]] == "usecond":
            dur_ms /= 1e3
        rd = val(r, "dram__bytes_read.sum", True) or 0.0
        wr = val(r, "dram__bytes_write.sum", True) or 0.0
        ks[name].append({"duration_ms": dur_ms, "dram_read_bytes": rd, "dram_write_bytes": wr,
                         "dram_gbs": (rd + wr) / (dur_ms / 1e3) / 1e9 if dur_ms else None,
                         "dram_pct_peak": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                         "registers": val(r, "launch__registers_per_thread"),
                         "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                         "grid": val(r, "launch__grid_size"),
                         # SM active / elapsed: below 1 = SMs idle for part of the kernel (tail, imbalance)
                         "sm_active_frac": (lambda a_, e_: a_ / e_ if a_ and e_ else None)(
                             val(r, "sm__cycles_active.avg") or val(r, "TPC.TriageCompute.sm__cycles_active.avg"),
                             val(r, "sm__cycles_elapsed.avg") or val(r, "gpc__cycles_elapsed.max"))})
    out = {}
    for k, v in ks.items():
        big = max(v, key=lambda x: x["dram_read_bytes"] + x["dram_write_bytes"])
        out[k] = {"launches": v, "dram_bytes_per_launch": big["dram_read_bytes"] + big["dram_write_bytes"],
                  "largest_launch": big}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--note", default="")
    ap.add_argument("--workload", default="cfg3", help="bench workload the capture was taken on")
    a = ap.parse_args()
    res = {"tag": a.tag, "note": a.note, "workload": a.workload}
    if a.launches:
        res["launch_list"] = launches(a.launches)
    if a.full:
        res["kernels"] = full(a.full)
    p = ROOT / "profiles" / f"{a.tag}_ncu_summary.json"
    p.write_text(json.dumps(res, indent=2) + "\n")
    print(p)
    print(json.dumps(res, indent=2)[:4000])


if __name__ == "__main__":
    main()
