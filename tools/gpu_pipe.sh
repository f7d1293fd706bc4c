#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_host_pipeline.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests_pipe.txt
timeout 400 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
