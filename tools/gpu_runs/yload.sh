#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/yl_res.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 > gpurun_out/pytest_gpu.log
for v in old new old new; do
  if [ $v = new ]; then lib=""; else lib="LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/y_$v.json 2>> gpurun_out/y.err
  python -c "import json; d=json.load(open('gpurun_out/y_$v.json')); print('$v', round(d['value'],1), d['spmv']['dsc_ms'], d['spmv']['wc_ms'])" >> gpurun_out/yl_res.log
done
