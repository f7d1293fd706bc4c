#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_mesh_device.py -m gpu -q 2>&1 | tail -2 > gpurun_out/gpu_tests_meshdev.txt
timeout 1500 python bench.py --fill 0.7 --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_fill_f32.json 2> gpurun_out/bench_fill_f32.err
timeout 1500 python bench.py --fill 0.7 --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype f64 > gpurun_out/bench_fill_f64.json 2> gpurun_out/bench_fill_f64.err
