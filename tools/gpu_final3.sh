#!/bin/bash
# round-end evidence refresh: full f32 bench (breakdown, nodal comparison, CPU baseline), full f64 bench,
# reference arm, ncu --set full of the fp64 N=9 stage kernel
mkdir -p gpurun_out; rm -f gpurun_out/prof* gpurun_out/bench_*
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --dtype f64 --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:opt_kernel -s 1 -c 1 -o gpurun_out/prof_stage_N9_f64 python tools/profile_kernel.py --N 9 --dtype f64 --op stage --reps 2 > gpurun_out/ncu_stage_N9_f64.log 2>&1
