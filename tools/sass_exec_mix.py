"""Executed-instruction mix of a kernel from an ncu report's SASS source page.

    python tools/sass_exec_mix.py rep.ncu-rep [units]

Prints warp instructions executed per opcode (and per `units` if given, e.g.
the number of warp-steps), plus the stall samples per opcode.
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
execd, stalls = Counter(), Counter()
total = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    opc = op[0] if not op[0].startswith("@") else op[1]
    opc = opc.split(".")[0]
    n = float(r[ix["Instructions Executed"]] or 0)
    execd[opc] += n
    stalls[opc] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    total += n
print("total warp instructions %.4g (%.2f per unit)" % (total, total / units))
for opc, n in execd.most_common(40):
    print("  %-10s %12.4g  %7.2f/unit  %5.1f%%  stall-samples %d" % (opc, n, n / units, 100 * n / total, stalls[opc]))
