for v in ${VARIANTS:-base keup kedn ng4 ng6}; do
  if [ $v = base ]; then L=""; else L="BBDG_LIB=variants/$v/libbbdg_cuda.so"; fi
  env $L timeout 600 python bench.py --quick --dtypes ${DT:-f32} --orders ${ORDERS:-4-9} --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tune_$v.json 2> gpurun_out/tune_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/tune_$v.json')); po=d['per_order']
print('$v', round(d['value'],1), ' '.join('%s:%.1f'%(N,po[N]['gdofs_stage']) for N in sorted(po)))"
done
