# ncu --set full of the first launch of kernel regex $2 on cfg3 (64 frames); report -> gpurun_out/$1.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:$2 -c 1 -o gpurun_out/$1 python tools/prof_step.py 3 64 2 > gpurun_out/ncu_$1.log 2>&1
tail -1 gpurun_out/ncu_$1.log
