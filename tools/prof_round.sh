#!/bin/bash
# Round profiling session (run under gpurun; one GPU): bench line, ncu launch list of a short
# bench run, and ncu --set full (with source) of each kernel on 64 cfg3 frames.  Every command
# runs once without ncu (and must exit 0) before it runs under ncu.  Then, locally:
#   python tools/save_profiles.py <tag>   (profiles/bench_<tag>.json, launches_<tag>.{csv,md},
#                                          ncu_summary_<tag>.{json,md}, ncu_lines_k{1,2}_<tag>.txt)
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log > gpurun_out/bench.json
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/plain_launch.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/prof_step.py 3 64 2 > gpurun_out/plain_step.log 2>&1 || exit 1
for k in k_ridges2:k1full k_rays:krays k_hough2:k2full k_fit:kfit; do
  re=${k%%:*}; name=${k##*:}
  ncu --set full --import-source on --clock-control none -k regex:$re -c 1 -o gpurun_out/$name \
      python tools/prof_step.py 3 64 2 > gpurun_out/ncu_$name.log 2>&1
  ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
done
