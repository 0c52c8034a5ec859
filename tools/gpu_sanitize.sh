#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every
# kernel variant (tools/sanitize_cases.py), one process per (tool, case).
# usage: bash tools/gpu_sanitize.sh TAG [cases...]
TAG=${1:-san}; shift
O=gpurun_out/$TAG
mkdir -p $O
CASES=${@:-$(python -c "import sys; sys.path.insert(0,'tools'); import sanitize_cases as s; print(' '.join(sorted(s.CASES)))")}
timeout 600 python tools/sanitize_cases.py > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/status.txt
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_cases.py $c > $O/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" >> $O/status.txt
  done
done
grep -h "ERROR SUMMARY" $O/*check_*.log | sort | uniq -c > $O/summary.txt
