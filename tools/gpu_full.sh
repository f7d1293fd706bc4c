#!/bin/bash
# full evidence run: bench (f32 full, f64 quick), reference arm, ncu captures, launch list
mkdir -p gpurun_out; rm -f gpurun_out/prof*
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --dtype f64 --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for cfg in "9 f32 stage" "3 f32 stage" "1 f32 stage" "9 f64 stage" "9 f32 volume" "9 f32 surface"; do set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tile_kernel|opt_kernel" -s 1 -c 1 -o gpurun_out/prof_$3_N$1_$2 python tools/profile_kernel.py --N $1 --dtype $2 --op $3 --reps 2 > gpurun_out/ncu_$3_N$1_$2.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
