#!/usr/bin/env python3
"""Summarise ncu output for profiles/ (run here, after gpurun brought the files back).

  python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/<round>_launches.md
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep [--traffic-json profiles/ncu_traffic.json --key quant_dar]

`launches`: the --metrics gpu__time_duration.sum launch list (cold-cache, serialised):
per-kernel-family launch counts, total and mean time and share of the listed time.
`full`: the --set full capture: duration, DRAM bytes (read + write) per launch,
throughput, IPC, occupancy, pipe utilisation, top stall reasons, instruction mix.
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys


def family(name: str) -> str:
    n = re.sub(r"\(.*", "", name.split("<")[0]).replace("void ", "").replace("dq::", "").strip()
    if n.startswith("k_quant"):
        tmpl = name[name.find("<") + 1:name.find(">")]
        parts = [p.strip() for p in tmpl.split(",")]
        dec = ",DEC" if len(parts) > 6 and parts[6] in ("1", "true") else ""
        return f"k_quant<NS={parts[0]},DAR={parts[3] if len(parts) > 3 else '?'}{dec}>"
    return n


def launches(path: str) -> None:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    fam = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
        f = family(r["Kernel Name"])
        fam[f][0] += 1
        fam[f][1] += ns
    tot = sum(v[1] for v in fam.values()) or 1.0
    print("| kernel family | launches | total µs | mean µs | share |")
    print("|---|---:|---:|---:|---:|")
    for f, (c, ns) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"| {f} | {c} | {ns / 1e3:.1f} | {ns / 1e3 / c:.1f} | {100 * ns / tot:.1f}% |")
    print(f"\n{sum(v[0] for v in fam.values())} launches, {tot / 1e3:.1f} µs listed (cold-cache, serialised).")


RAW_KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "pipe_fmaheavy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
}


def full(path: str, traffic_json=None, key=None) -> None:
    if path.endswith(".csv"):  # an exported raw page (tools/ncu_export.sh)
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")]}
        for k, name in RAW_KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(d[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if name.startswith("dram_r") or name.startswith("dram_w"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if name == "duration":
                    v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1}.get(u, 1)
                rec[name] = v
        stalls = {h.split("stalled_")[1].split("_per")[0]: float(d[i])
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                  and d[i] not in ("", "n/a")}
        rec["top_stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        out.append(rec)
    print("| kernel | µs | DRAM MB (r+w) | DRAM GB/s | issue active | IPC-ish | ALU pipe | FMA pipe | occupancy | regs | top stalls (warps/issue) |")
    print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|")
    for r in out:
        dram = r.get("dram_read", 0) + r.get("dram_write", 0)
        us = r.get("duration", 0)
        ipc = r.get("inst_executed", 0) / max(us * 1e-6 * 1.965e9 * 148, 1)  # warp-instr / SM / cycle at max clock
        st = ", ".join(f"{k} {v:.2f}" for k, v in r["top_stalls"])
        print(f"| {r['kernel'][:60]} | {us:.1f} | {dram / 1e6:.1f} | {dram / max(us, 1e-9) / 1e3:.0f} | "
              f"{r.get('issue_active_pct', 0):.0f}% | {ipc:.2f} | {r.get('pipe_alu_pct', 0):.0f}% | "
              f"{r.get('pipe_fma_pct', 0):.0f}% | {r.get('occupancy_pct', 0):.0f}% | {r.get('registers', 0):.0f} | {st} |")
    if traffic_json and key and out:
        try:
            j = json.load(open(traffic_json))
        except Exception:
            j = {}
        r = out[0]
        j[key] = {"dram_bytes_per_launch": r.get("dram_read", 0) + r.get("dram_write", 0),
                  "duration_us_cold": r.get("duration"), "kernel": r["kernel"], "source": path}
        json.dump(j, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else None
        full(sys.argv[2], tj, key)
