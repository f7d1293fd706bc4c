#!/bin/bash
cd /root/repo/gpurun_out
tail -3 gpu_tests.txt
for f in bench_quick.json bench_quick64.json; do python3 -c "
import json,sys; d=json.load(open('$f'))
print('$f value', round(d['value'],2), round(d['roofline']['frac'],3), [round(r['gdofs_stage'],1) for N,r in d['per_order'].items()])
" 2>/dev/null || tail -3 ${f%.json}.err; done
for f in prof_stage_N9_f32 prof_stage_N3_f32 prof_stage_N6_f32; do [ -f $f.ncu-rep ] || continue; echo "== $f"; python3 /root/repo/tools/ncu_summary.py $f.ncu-rep | grep -E "time|dram_thr|issue_active|warps_active|bank|registers|inst_executed.sum|wavefronts"; ncu -i $f.ncu-rep --page source --csv --print-source cuda,sass > /tmp/s_$f.csv 2>/dev/null; python3 /root/repo/tools/ncu_phases.py /tmp/s_$f.csv /root/repo/paper_1512_06025_b200/csrc/bbdg_tile.cuh; done
