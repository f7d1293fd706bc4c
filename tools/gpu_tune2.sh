#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nodal > gpurun_out/tune_full_default.json 2> gpurun_out/tune_full_default.err
BBDG_LIB=$PWD/variants/vS/libbbdg_cuda.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nodal > gpurun_out/tune_full_vS.json 2> gpurun_out/tune_full_vS.err
