# per-launch DRAM bytes of one hot-path kernel on the bench's HBM-filling boxes (one order per call):
#   bash tools/fill_traffic_capture.sh <dtype> <N> <nx,ny,nz> <xblock> [op: stage|volume|surface|update]
OP=${5:-stage}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
SUF=$([ "$OP" = stage ] && echo "" || echo "_$OP")
timeout 900 ncu --metrics $M --clock-control none -k regex:"opt_kernel|ept_kernel|lsrk_update" -s 1 -c 1 --csv \
  --log-file gpurun_out/fill_traffic_$1_$2$SUF.csv python tools/profile_kernel.py --N $2 --dtype $1 --op $OP \
  --box $3 --xblock $4 --reps 2 > /dev/null 2>&1
grep -h "dram__bytes\|gpu__time" gpurun_out/fill_traffic_$1_$2$SUF.csv | cut -d, -f12-16
