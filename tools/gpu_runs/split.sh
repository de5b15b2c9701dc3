#!/bin/bash
mkdir -p gpurun_out
LIFE_B200_LIB=$PWD/build/split/liblife_b200.so timeout 300 python tools/tc_check.py --c1 > gpurun_out/split_c1.log 2>&1
for v in base split base split; do
  if [ $v = base ]; then lib=""; else lib="LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/s_$v.json 2>> gpurun_out/s.err
  python -c "import json; d=json.load(open('gpurun_out/s_$v.json')); print('$v', round(d['value'],1), d['spmv']['dsc_ms'], d['spmv']['wc_ms'])" >> gpurun_out/split_res.log
done
