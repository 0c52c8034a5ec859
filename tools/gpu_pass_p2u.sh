#!/bin/bash
# cfg3 n=256: register vs shared-constant (tight) J=16 layouts, alternating, pinned via SDEB200_LAYOUT
TAG=${1:-p2u}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2 3; do
  for lay in 16,1,0,0 16,0,0,0 16,1,0,1 16,0,0,1; do
    SDEB200_LAYOUT=$lay timeout 300 python bench.py --workload cfg3_n256 --no-cold --no-secondary --no-cpu-baseline --steps 10 > $O/b_${lay//,/_}_$r.log 2>&1
    python -c "
import json
l=[x for x in open('$O/b_${lay//,/_}_$r.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$lay', $r, '%.4g'%d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/table.txt 2>&1
  done
done
