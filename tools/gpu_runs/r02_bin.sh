#!/bin/bash
# binned products: accuracy/timing sweep (incl. C2) and the C2 launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python tools/bin_check.py --c2 ${LAYOUTS:+--layouts $LAYOUTS} > gpurun_out/bin_check.log 2>&1
tail -20 gpurun_out/bin_check.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_side|k_tile|k_wc_fin" --csv \
    --log-file gpurun_out/bin_launch.csv python tools/bin_prof.py > gpurun_out/bin_prof.log 2>&1
python tools/launch_summary.py gpurun_out/bin_launch.csv "# C2 bin launch list" > gpurun_out/bin_launch.txt
cat gpurun_out/bin_launch.txt
