#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/tune_*
timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype f64 > gpurun_out/tune_default.json 2> gpurun_out/tune_default.err
for v in variants/*/; do n=$(basename $v)
  BBDG_LIB=$PWD/variants/$n/libbbdg_cuda.so timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype f64 > gpurun_out/tune_$n.json 2> gpurun_out/tune_$n.err
done
