#!/bin/bash
# quick stage sweep for the default library and every built tuning variant (f64 variants: names ending in d)
mkdir -p gpurun_out; rm -f gpurun_out/tune_*
timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/tune_default.json 2> gpurun_out/tune_default.err
timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype f64 > gpurun_out/tune_default_d.json 2> gpurun_out/tune_default_d.err
for v in variants/*/; do n=$(basename $v); dt=f32; [[ $n == *d ]] && dt=f64
  BBDG_LIB=$PWD/variants/$n/libbbdg_cuda.so timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype $dt > gpurun_out/tune_$n.json 2> gpurun_out/tune_$n.err
done
