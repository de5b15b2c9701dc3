#!/bin/bash
# staging chunk / thread sweep of the host-input construction at C2 (tools/setup_time.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "16384 12" "1024 12" "512 12" "256 12" "1024 16" "256 16" "4096 12"; do
  set -- $cfg
  echo "== chunk ${1} KB, ${2} threads"
  LIFE_B200_STAGE_KB=$1 LIFE_B200_STAGE_THREADS=$2 timeout 300 python tools/setup_time.py 2>&1 | grep -v "^\[life" | tail -6
done
