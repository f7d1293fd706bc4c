#!/bin/bash
# full evidence run: bench (f32, f64), reference arm, 2 ncu captures, launch list, per-order DRAM traffic
# (gpurun copies back at most 64 MiB: a --set full report is ~14 MB; more captures via tools/gpu_ncu.sh)
mkdir -p gpurun_out; rm -f gpurun_out/prof* gpurun_out/traffic_*.csv
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --dtype f64 --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for cfg in ${PROFS:-"9 f32 stage" "9 f64 stage"}; do set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"opt_kernel|tile_kernel" -s 1 -c 1 -o gpurun_out/prof_$3_N$1_$2 python tools/profile_kernel.py --N $1 --dtype $2 --op $3 --reps 2 > gpurun_out/ncu_$3_N$1_$2.log 2>&1
done
for dt in f32 f64; do for N in 1 2 3 4 5 6 7 8 9; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:opt_kernel -s 1 -c 1 --csv --log-file gpurun_out/traffic_${dt}_N${N}.csv python tools/profile_kernel.py --N $N --dtype $dt --n 40 --reps 2 > /dev/null 2>&1
done; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
