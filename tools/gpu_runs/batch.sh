#!/bin/bash
mkdir -p gpurun_out
for v in ${VARIANTS:-base fb3 fb2 sr4 fb3sr4}; do
  if [ $v = base ]; then lib=""; else lib="LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/b_$v.json 2>> gpurun_out/b.err
done
