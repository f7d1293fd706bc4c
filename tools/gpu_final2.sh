#!/bin/bash
# round-end evidence: full bench f32 (per-kernel breakdown, nodal comparison, CPU baseline), f64, reference arm,
# the ncu launch list of a short bench run, and one ncu --set full capture of the N=9 fp32 stage kernel
mkdir -p gpurun_out; rm -f gpurun_out/prof* gpurun_out/bench_*
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --dtype f64 --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline --orders 1-8 > gpurun_out/bench_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:opt_kernel -s 1 -c 1 -o gpurun_out/prof_stage_N9_f32 python tools/profile_kernel.py --N 9 --dtype f32 --op stage --reps 2 > gpurun_out/ncu_stage_N9_f32.log 2>&1
