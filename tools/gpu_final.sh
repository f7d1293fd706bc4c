#!/bin/bash
# final evidence run (gpurun copies back <= 64 MiB: one ncu --set full report)
mkdir -p gpurun_out; rm -f gpurun_out/prof* gpurun_out/traffic_*.csv
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --dtype f64 --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1500 python bench.py --fill 0.7 --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_fill_f32.json 2> gpurun_out/bench_fill_f32.err
for dt in f32 f64; do for N in 1 2 3 4 5 6 7 8 9; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:opt_kernel -s 1 -c 1 --csv --log-file gpurun_out/traffic_${dt}_N${N}.csv python tools/profile_kernel.py --N $N --dtype $dt --n 40 --reps 2 > /dev/null 2>&1
done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:opt_kernel -s 1 -c 1 -o gpurun_out/prof_stage_N9_f32 python tools/profile_kernel.py --N 9 --dtype f32 --op stage --reps 2 > gpurun_out/ncu_stage_N9_f32.log 2>&1
