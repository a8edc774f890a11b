#!/bin/bash
# A/B timing of library variants (run under gpurun): tools/ab_run.sh cfg frames reps lib1.so lib2.so ...
# Each variant's per-kernel us/frame (tools/cap_probe.py), interleaved over reps rounds.
cfg=$1; n=$2; reps=$3; shift 3
for r in $(seq 1 $reps); do
  for lib in "$@"; do
    echo -n "$(basename $lib) "
    RD_LIB_PATH=$PWD/$lib python tools/cap_probe.py $cfg $n 2>&1 | grep "us/frame"
  done
done
