#!/usr/bin/env python
"""Top SASS lines by warp-stall samples from an ncu report's source page.
usage: python profiles/ncu_hot.py REPORT KERNEL_REGEX SKIP [TOP]"""
import csv
import io
import subprocess
import sys

rep, rx, skip = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}", "--launch-skip",
                      skip, "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc, iss, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
data = [(int(r[iss] or 0), int(r[ie] or 0), r[isrc].strip(), k) for k, r in enumerate(rows[1:])
        if len(r) > max(iss, ie, isrc) and r[iss].isdigit() and r[ie].isdigit()]
tot = sum(d[0] for d in data)
tot_i = sum(d[1] for d in data)
print(f"samples {tot}  warp-instructions {tot_i}")
for s, e, src, k in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}%  {e:9d}  [{k:5d}] {src}")
