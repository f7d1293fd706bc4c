#!/bin/bash
# verification of the current tree: gpu tests, smoke, quick f32/f64 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
timeout 400 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --dtype f64 > gpurun_out/bench_quick64.json 2> gpurun_out/bench_quick64.err
