#!/usr/bin/env python3
"""Per-source-line dynamic instruction counts of one kernel: joins an ncu SASS source page
(CSV, per-instruction 'Instructions Executed') with the line table of the same cubin
(nvdisasm -g).  Usage: sass_lines.py <cubin> <mangled-kernel> <ncu_sass.csv[.gz]> [top]"""
import csv, gzip, io, re, subprocess, sys
from collections import defaultdict

cubin, fn, page = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = dis.split(f".text.{fn}:")[1].split("//--------------------- .text.")[0]
lines, cur = [], None
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", ln):
        lines.append((cur, ln.split("*/", 1)[1].strip().rstrip(";").strip()))
op = gzip.open(page, "rt") if page.endswith(".gz") else open(page)
rows = list(csv.reader(op))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > ie]
if len(data) != len(lines):
    print(f"warning: {len(data)} profiled vs {len(lines)} disassembled instructions", file=sys.stderr)
per, opc = defaultdict(int), defaultdict(int)
total = 0
for (src, ins), r in zip(lines, data):
    n = int(r[ie] or 0)
    per[src] += n
    o = re.sub(r"^@!?U?P\w+\s+", "", ins).split()[0].split(".")[0] if ins else "?"
    opc[o] += n
    total += n
print(f"total warp-instructions executed: {total}")
for k, v in sorted(per.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:>12} {100 * v / total:5.1f}%  {k}")
print("-- by opcode")
for k, v in sorted(opc.items(), key=lambda x: -x[1])[:30]:
    print(f"{v:>12} {100 * v / total:5.1f}%  {k}")
