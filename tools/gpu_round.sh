#!/bin/bash
# GPU tests, sensitivity study, and the tuning variants' quick sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gpu_tests.txt
timeout 900 python tools/sensitivity.py --out gpurun_out/sensitivity.json > gpurun_out/sensitivity.txt 2>&1
bash tools/gpu_tune.sh
