#!/bin/bash
# binned products: accuracy/timing sweep (incl. C2 and the skew cases) and
# the C2 / C2-Zipf launch lists
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python tools/bin_check.py --c2 ${LAYOUTS:+--layouts $LAYOUTS} > gpurun_out/bin_check.log 2>&1
tail -20 gpurun_out/bin_check.log
if [ "${SKEW:-1}" = 1 ]; then
  timeout 1200 python tools/bin_check.py --skew > gpurun_out/bin_skew.log 2>&1
  cat gpurun_out/bin_skew.log
fi
for z in ${CASES:-"" --zipf}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_side|k_tile|k_wc_fin" --csv \
      --log-file gpurun_out/bin_launch$z.csv python tools/bin_prof.py $z > gpurun_out/bin_prof$z.log 2>&1
  python tools/launch_summary.py gpurun_out/bin_launch$z.csv "# C2$z bin launch list" > gpurun_out/bin_launch$z.txt
  cat gpurun_out/bin_launch$z.txt
done
