#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/prof* gpurun_out/launches*.csv
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline --n 26 > gpurun_out/bench_under_ncu.log 2>&1
bash tools/gpu_ncu.sh
