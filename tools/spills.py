#!/usr/bin/env python3
"""List kernels with spills / stack frames from the ptxas -v logs of the library build."""
import glob, re, subprocess, sys
rows = []
for log in sorted(glob.glob("/root/repo/paper_2602_08923_b200/csrc/build/*.ptxas.log")):
    fn = None
    for ln in open(log):
        m = re.search(r"Compiling entry function '(\w+)'", ln)
        if m:
            fn = m.group(1)
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m and fn:
            st, ss, sl = map(int, m.groups())
            if st or ss or sl or "-a" in sys.argv:
                rows.append((fn, st, ss, sl))
        m = re.search(r"Used (\d+) registers", ln)
        if m and fn and rows and rows[-1][0] == fn and len(rows[-1]) == 4:
            rows[-1] = rows[-1] + (int(m.group(1)),)
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
for r, n in zip(rows, names):
    print(f"stack {r[1]:3} spill st {r[2]:3} ld {r[3]:3} regs {r[4] if len(r) > 4 else '?':>3}  {n[:150]}")
