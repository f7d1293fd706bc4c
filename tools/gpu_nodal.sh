#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "nodal" 2>&1 | tail -15 > gpurun_out/gpu_tests_nodal.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
timeout 600 python tools/nodal_timing.py > gpurun_out/nodal_timing.txt 2>&1
