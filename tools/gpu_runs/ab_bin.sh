#!/bin/bash
# A/B of binned-product build variants (build/<name>/liblife_b200.so) on the
# bin_check shapes incl. C2: accuracy vs fp64, repeatability, DSC/WC times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in default "$@"; do
  echo "== $v"
  if [ "$v" = default ]; then lib=""; else lib="build/$v/liblife_b200.so"; fi
  LIFE_B200_LIB=$lib timeout 600 python tools/bin_check.py --c2 2>&1 | tail -12
done
