#!/bin/bash
# one GPU iteration: gpu tests, quick f32/f64 bench, ncu full of the N=9 and N=3 f32 stage kernels
mkdir -p gpurun_out; rm -f gpurun_out/prof*
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype f64 > gpurun_out/bench_quick64.json 2> gpurun_out/bench_quick64.err
for cfg in "9 f32" "3 f32" "6 f32"; do set -- $cfg; timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tile_kernel|opt_kernel" -s 1 -c 1 -o gpurun_out/prof_stage_N$1_$2 python tools/profile_kernel.py --N $1 --dtype $2 --op stage --reps 2 > gpurun_out/ncu_N$1_$2.log 2>&1; done
