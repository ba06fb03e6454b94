#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/ncu_summary.py --round r01 \
        --full c3:match_tc:gpurun_out/prof_c3.ncu-rep \
        --full c3:match_tc_scan:gpurun_out/prof_scan.ncu-rep \
        --launches c3:gpurun_out/launches_c3.csv

Writes profiles/ncu_summary.json ({workload: {kernel: {...metrics, dram_bytes_per_launch}}},
read by bench.py for roofline.traffic when build_id matches the library it runs),
profiles/ncu_<round>_<workload>_<kernel>.txt
(raw key metrics) and profiles/launches_<round>_<workload>.csv (+ a per-kernel share
table).  Runs here (no GPU needed): `ncu -i` only reads the report files.
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__shared_mem_per_block_dynamic", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
              "nsecond": 1e-9}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            m[h] = {"value": x, "unit": u}
    return m


def to_base(entry):
    return entry["value"] * UNIT_SCALE.get(entry["unit"], 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--full", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--build-id-file", default=None,
                    help="ams_build_id() of the library the capture ran, written on the GPU box by the capture "
                         "command; bench.py reuses a capture's traffic only for that build")
    a = ap.parse_args()
    build_id = open(a.build_id_file).read().split()[0] if a.build_id_file else None
    os.makedirs(PROF, exist_ok=True)
    path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for spec in a.full:
        wl, kname, rep = spec.split(":", 2)
        m = raw_metrics(rep)
        rd = to_base(m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_base(m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        entry = {"round": a.round, "report": os.path.basename(rep), "build_id": build_id,
                 "dram_bytes_per_launch": (rd + wr) if rd is not None and wr is not None else None,
                 "duration_s": to_base(m["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in m else None,
                 "metrics": {k: v["value"] for k, v in m.items()},
                 "units": {k: v["unit"] for k, v in m.items()}}
        summary.setdefault(wl, {})[kname] = entry
        with open(os.path.join(PROF, f"ncu_{a.round}_{wl}_{kname}.txt"), "w") as f:
            for k in KEYS:
                if k in m:
                    f.write(f"{k:90s} {m[k]['value']:>18.6g} {m[k]['unit']}\n")
        shutil.copy(rep, os.path.join(PROF, f"ncu_{a.round}_{wl}_{kname}.ncu-rep"))
    for spec in a.launches:
        wl, f = spec.split(":", 1)
        dst = os.path.join(PROF, f"launches_{a.round}_{wl}.csv")
        shutil.copy(f, dst)
        text = open(f).read()
        start = text.find('"ID"')
        rows = list(csv.DictReader(io.StringIO(text[start:])))
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
            name = name.split("(")[0].split("<")[0]
            name = name.replace("void ", "")
            x = float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r["Metric Unit"], 1.0)
            tot[name] += x
            cnt[name] += 1
        allt = sum(tot.values()) or 1.0
        with open(os.path.join(PROF, f"launches_{a.round}_{wl}_share.txt"), "w") as fo:
            fo.write(f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'avg_ms':>10s} {'share':>7s}\n")
            for k in sorted(tot, key=lambda x: -tot[x]):
                fo.write(f"{k:40s} {cnt[k]:8d} {tot[k]*1e3:10.3f} {tot[k]/cnt[k]*1e3:10.4f} {tot[k]/allt:7.1%}\n")
        summary.setdefault(wl, {})["_launch_shares"] = {k: tot[k] / allt for k in tot}
    with open(path, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({w: {k: (v.get("dram_bytes_per_launch") if isinstance(v, dict) else None)
                          for k, v in d.items()} for w, d in summary.items()}, indent=1))


if __name__ == "__main__":
    main()
