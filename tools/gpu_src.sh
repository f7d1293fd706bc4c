#!/bin/bash
# source-level ncu captures of the fused stage (N=9 and N=6 fp32) for per-line wavefront attribution
mkdir -p gpurun_out; rm -f gpurun_out/prof*
for cfg in "9 f32 stage" "6 f32 stage" "9 f32 surface"; do set -- $cfg
timeout 300 ncu --set full --clock-control none --import-source on -k regex:opt_kernel -s 1 -c 1 -o gpurun_out/prof_$3_N$1_$2 python tools/profile_kernel.py --N $1 --dtype $2 --op $3 --reps 2 > gpurun_out/ncu_$3_N$1_$2.log 2>&1
done
