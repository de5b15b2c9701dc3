#!/bin/bash
# ncu --set full of the bin-side kernels, C2 uniform vs Zipf fascicles
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for z in "" --zipf; do
  for k in k_side_dsc k_side_wc; do
    timeout 900 ncu --set full --clock-control none --import-source on -k $k --launch-skip 1 -c 1 \
        -o gpurun_out/ncu_${k}${z} -f python tools/bin_prof.py $z > gpurun_out/ncu_${k}${z}.log 2>&1
    tail -2 gpurun_out/ncu_${k}${z}.log
  done
done
ls -la gpurun_out/*.ncu-rep
