#!/usr/bin/env python
"""Summarize ncu outputs brought back in gpurun_out/ into profiles/.

  python scripts/ncu_summarize.py TAG [--launches gpurun_out/launches_TAG.csv]
                                      [--rep gpurun_out/pass_TAG.ncu-rep]
                                      [--m 10000 --n 10000 --dtype f32]

Writes profiles/TAG_launches.md (per-kernel device-time share of the launch
list: cold-cache, serialized -- shares, not absolutes), profiles/TAG_pass.md
(key metrics of the full capture of the fused sweep) and updates
profiles/ncu_pass_summary.json (DRAM bytes per sweep launch, read by bench.py
as roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("void ", "")
    return name[:90]


def read_csv_after_header(path):
    with open(path, errors="replace") as f:
        lines = f.read().splitlines()
    for k, ln in enumerate(lines):
        if ln.startswith('"ID"'):
            return list(csv.DictReader(io.StringIO("\n".join(lines[k:]))))
    return []


def launches(path, tag):
    rows = read_csv_after_header(path)
    per = defaultdict(lambda: [0, 0.0])
    unit = "ns"
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", unit)
        v = float(r["Metric Value"].replace(",", ""))
        k = short(r["Kernel Name"])
        per[k][0] += 1
        per[k][1] += v
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(v[1] for v in per.values()) or 1.0
    out = [f"# {tag}: ncu launch list ({os.path.basename(path)})", "",
           "Cold-cache, serialized replay (`--metrics gpu__time_duration.sum "
           "--clock-control none`): compare shares, not absolute times.", "",
           "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {c} | {v * scale:.1f} | {v * scale / c:.2f} | {100 * v / tot:.1f}% |")
    return "\n".join(out) + "\n", per, scale


RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes.sum.per_second",
]


def full_capture(rep, tag, alg_bytes):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                       text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return None, None
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: k for k, h in enumerate(hdr)}
    launches_ = []
    for d in data:
        e = {"kernel": short(d[idx["Kernel Name"]])}
        for key in RAW_KEYS:
            if key in idx:
                e[key] = d[idx[key]]
                e[key + ".unit"] = units[idx[key]]
        launches_.append(e)
    out = [f"# {tag}: ncu --set full of the fused sweep ({os.path.basename(rep)})", ""]
    for e in launches_:
        out.append(f"## `{e['kernel']}`")
        out.append("")
        out.append("| metric | value | unit |")
        out.append("|---|---|---|")
        for key in RAW_KEYS:
            if key in e:
                out.append(f"| {key} | {e[key]} | {e[key + '.unit']} |")
        try:
            rd = float(e["dram__bytes_read.sum"].replace(",", ""))
            wr = float(e["dram__bytes_write.sum"].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= mult.get(e["dram__bytes_read.sum.unit"], 1)
            wr *= mult.get(e["dram__bytes_write.sum.unit"], 1)
            e["dram_bytes"] = rd + wr
            if alg_bytes:
                out.append(f"| DRAM traffic / algorithmic bytes | {(rd + wr) / alg_bytes:.3f} | "
                           f"({rd + wr:.4g} / {alg_bytes:.4g}) |")
        except Exception:
            pass
        out.append("")
    return "\n".join(out) + "\n", launches_


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--m", type=int, default=10000)
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--key", default=None, help="summary key prefix (default pass / solve)")
    ap.add_argument("--iters-per-launch", type=int, default=0,
                    help="persistent solve_kernel capture: iterations per launch "
                         "(alternating fold / skip sweeps)")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    go = os.path.join(ROOT, "gpurun_out")
    lpath = args.launches or os.path.join(go, f"launches_{args.tag}.csv")
    rpath = args.rep or os.path.join(go, f"pass_{args.tag}.ncu-rep")
    s = 4 if args.dtype == "f32" else 8
    if os.path.exists(lpath):
        md, per, scale = launches(lpath, args.tag)
        with open(os.path.join(PROF, f"{args.tag}_launches.md"), "w") as f:
            f.write(md)
        print(md)
    if os.path.exists(rpath):
        md, ls = full_capture(rpath, args.tag, None)
        if md:
            # algorithmic bytes: fold/plain sweeps 3*s*m*n, skip sweeps 2*s*m*n
            for e in ls:
                if args.iters_per_launch:
                    k = args.iters_per_launch
                    e["algorithmic_bytes"] = (3 * ((k + 1) // 2) + 2 * (k // 2)) * s * args.m * args.n
                    continue
                skip = re.search(r"<(float|double), 3,", e["kernel"]) is not None
                e["algorithmic_bytes"] = (2 if skip else 3) * s * args.m * args.n
            md2, _ = full_capture(rpath, args.tag, None)
            lines = [md2]
            for e in ls:
                if "dram_bytes" in e:
                    lines.append(f"- `{e['kernel']}`: DRAM {e['dram_bytes'] / 1e9:.4f} GB vs "
                                 f"algorithmic {e['algorithmic_bytes'] / 1e9:.4f} GB "
                                 f"(ratio {e['dram_bytes'] / e['algorithmic_bytes']:.3f})")
            with open(os.path.join(PROF, f"{args.tag}_pass.md"), "w") as f:
                f.write("\n".join(lines) + "\n")
            print("\n".join(lines))
            sp = os.path.join(PROF, "ncu_pass_summary.json")
            summ = {}
            if os.path.exists(sp):
                with open(sp) as f:
                    summ = json.load(f)
            dram = [e["dram_bytes"] for e in ls if "dram_bytes" in e]
            if dram:
                key = (args.key or ("solve" if args.iters_per_launch else "pass")) + \
                    f"_{args.m}x{args.n}_{args.dtype}"
                summ[key] = {
                    "tag": args.tag,
                    "dram_bytes_per_launch_avg": sum(dram) / len(dram),
                    "iters_per_launch": args.iters_per_launch or None,
                    "dram_bytes_per_iteration": (sum(dram) / len(dram) / args.iters_per_launch)
                    if args.iters_per_launch else None,
                    "launches": [{"kernel": e["kernel"], "dram_bytes": e.get("dram_bytes"),
                                  "algorithmic_bytes": e["algorithmic_bytes"]} for e in ls],
                }
                with open(sp, "w") as f:
                    json.dump(summ, f, indent=1)


if __name__ == "__main__":
    main()
