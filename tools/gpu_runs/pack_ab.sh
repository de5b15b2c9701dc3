#!/bin/bash
# A/B of the packed atom+voxel transfer (LIFE_B200_NO_PACK=1 disables it), alternating runs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do
  for np in 0 1; do
    echo "== LIFE_B200_NO_PACK=$np (round $r)"
    LIFE_B200_NO_PACK=$np timeout 300 python tools/setup_time.py 2>&1 | grep -v "^\[life" | tail -6
  done
done
