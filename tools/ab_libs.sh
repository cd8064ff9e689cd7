#!/bin/bash
# Same-box A/B of two builds: libffb200_old.so (repo root) vs the in-tree
# library, interleaved processes, `perf_probe.py --sets calib_mask=15` (3
# timings each).  usage: tools/ab_libs.sh REPS "<perf_probe args>" ...
REPS=$1; shift
for args in "$@"; do
  for r in $(seq $REPS); do
    for L in old new; do
      if [ $L = old ]; then export FFB200_LIB=$PWD/libffb200_old.so; else unset FFB200_LIB; fi
      echo "== $L $args"
      timeout 300 python tools/perf_probe.py --calibrate 8 --steps 100 $args --sets "calib_mask=15" 2>&1 | grep -v calibrated
    done
  done
done
