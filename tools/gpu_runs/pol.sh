#!/bin/bash
mkdir -p gpurun_out
for v in base pol_s0 pol_k0 pol_s0k0 pol_s3; do
  if [ $v = base ]; then lib=""; else lib="LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so"; fi
  env $lib timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/pol_$v.json 2>> gpurun_out/pol.err
done
