#!/bin/bash
# late round 2: ncu --set full of the changed WC kernels at C2 (992-unit
# chunks, Z ring of 3) and the launch list of the default bench command
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for k in k_tile_wc k_side_wc; do
  timeout 900 ncu --set full --clock-control none --import-source on -k $k --launch-skip 2 -c 1 \
      -o gpurun_out/r02b_${k} -f python tools/bin_prof.py > gpurun_out/r02b_${k}.log 2>&1
  tail -1 gpurun_out/r02b_${k}.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02b_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/r02b_bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r02b_bench_launches.csv "# launch list: ncu --metrics gpu__time_duration.sum python bench.py --steps 2 --warmup 3 (C2, late round 2)" > gpurun_out/r02b_bench_launches.txt
head -30 gpurun_out/r02b_bench_launches.txt
