"""Summarise `ptxas -v` output of the build: kernel -> registers, spills."""
import re
import subprocess
import sys

out = subprocess.run([sys.executable, "-m", "paper_1908_03869_b200._build", "-v", "--force"],
                     capture_output=True, text=True).stdout
cur = None
rows = []
for ln in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        spill = None
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur:
        rows.append((cur, int(m.group(1)), spill))
        cur = None
pat = sys.argv[1] if len(sys.argv) > 1 else "kuramoto_run"
for name, regs, spill in rows:
    if pat in name:
        t = re.search(r"ILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)EL[ib](\d)E", name)
        tag = ("J=%s solver=%s stream=%s coupling=%s variant=%s" % t.groups()) if t else name
        print("%-45s regs %3d spill %s" % (tag, regs, spill))
