# per-launch DRAM bytes of the fused stage on the bench's HBM-filling boxes (one order per call):
#   bash tools/fill_traffic_capture.sh <dtype> <N> <nx,ny,nz> <xblock>
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"opt_kernel|ept_kernel" -s 1 -c 1 --csv \
  --log-file gpurun_out/fill_traffic_$1_$2.csv python tools/profile_kernel.py --N $2 --dtype $1 --op stage \
  --box $3 --xblock $4 --reps 2 > /dev/null 2>&1
grep -h "dram__bytes\|gpu__time" gpurun_out/fill_traffic_$1_$2.csv | cut -d, -f12-16
