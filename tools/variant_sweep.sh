#!/bin/bash
# Compare library variants (tools/build_variant.py) on pinned layouts.
# usage: bash tools/variant_sweep.sh TAG "variant ..." "workload:layouts ..."
TAG=$1; VARS=$2; JOBS=$3
O=gpurun_out/$TAG
mkdir -p $O
for v in base $VARS; do
  if [ "$v" = "base" ]; then LIB=$PWD/paper_1908_03869_b200/libsdeb200.so; else LIB=$PWD/paper_1908_03869_b200/_variants/$v/libsdeb200.so; fi
  for job in $JOBS; do
    wl=${job%%:*}; lays=${job#*:}
    SDEB200_LIB=$LIB timeout 600 python tools/layout_sweep.py --workload $wl --layouts "$lays" > $O/${v}_$wl.log 2>&1
  done
done
