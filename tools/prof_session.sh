#!/bin/bash
# One GPU profiling session (run under gpurun): bench line, phase cycles of K2 (prof build),
# ncu --set full with source of K1 and K2 (64 cfg3 frames), source pages as CSV.
# usage: tools/prof_session.sh TAG
TAG=${1:-x}
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log > gpurun_out/bench_$TAG.json
RD_LIB_PATH=variants/librd_prof.so python tools/phase_probe.py 3 128 > gpurun_out/phase_$TAG.log 2>&1
for k in k_hough2 k_ridges2 k_rays; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${k}_$TAG python tools/prof_step.py 3 64 2 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  ncu -i gpurun_out/${k}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${k}_${TAG}_src.csv 2>/dev/null
done
ncu -i gpurun_out/k_hough2_$TAG.ncu-rep --page raw --csv > gpurun_out/k_hough2_${TAG}_raw.csv 2>/dev/null
