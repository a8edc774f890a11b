#!/bin/bash
# tools-like A/B over env settings: ab_env.sh cfg n reps "ENV=.." "ENV=.."
cfg=$1; n=$2; reps=$3; shift 3
for r in $(seq 1 $reps); do for e in "$@"; do echo -n "$e "; env $e python tools/cap_probe.py $cfg $n 2>&1 | grep "us/frame"; done; done
