#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-base tcu1 tcu2}; do
  if [ $v = base ]; then lib=""; else lib="LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 60 --warmup 5 --no-cpu --no-e2e --layout tensor > gpurun_out/t_$v.json 2>> gpurun_out/t.err
done
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/qb.json 2>> gpurun_out/t.err
