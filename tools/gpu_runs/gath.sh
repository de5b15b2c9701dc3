#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/g_res.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 > gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-base g4 g5 g6 g8}; do
  if [ $v = base ]; then lib=""; else lib="LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/g_$v.json 2>> gpurun_out/g.err
  python -c "import json; d=json.load(open('gpurun_out/g_$v.json')); print('$v', round(d['value'],1), d['spmv']['dsc_ms'], d['spmv']['wc_ms'])" >> gpurun_out/g_res.log
done
