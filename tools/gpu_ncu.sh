#!/bin/bash
# ncu --set full captures (3 per call: gpurun copies back <= 64 MiB)
mkdir -p gpurun_out; rm -f gpurun_out/prof*
for cfg in ${PROFS:-"5 f32 stage" "9 f32 volume" "9 f32 surface"}; do set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"opt_kernel|tile_kernel|nodal_mma" -s 1 -c 1 -o gpurun_out/prof_$3_N$1_$2 python tools/profile_kernel.py --N $1 --dtype $2 --op $3 --reps 2 ${4:+--basis $4} ${5:+--lift $5} > gpurun_out/ncu_$3_N$1_$2.log 2>&1
done
