"""Count SASS opcodes inside the innermost hot loop of a kernel (by backward branch)."""
import re
import sys
from collections import Counter

path, = sys.argv[1:2]
lines = open(path).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, text) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?(0x[0-9a-f]+)", text)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a:
            loops.append((tgt, a))
loops.sort(key=lambda t: t[1] - t[0], reverse=True)
for lo, hi in loops[:6]:
    body = [t for a, t in ins if lo <= a <= hi]
    ops = Counter()
    for t in body:
        op = re.sub(r"^@!?U?P[T\d]\s+", "", t).split()[0].split(".")[0]
        ops[op] += 1
    fp64 = sum(ops[o] for o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
    print("loop 0x%x-0x%x: %d instr, fp64 %d" % (lo, hi, len(body), fp64))
    print("   ", ", ".join("%s %d" % kv for kv in ops.most_common(22)))
