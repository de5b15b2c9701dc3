#!/bin/bash
# tile count rounded to a multiple of the tile grid (default) vs full tiles
# only (LIFE_B200_NO_TILE_ROUND=1): C2 and the 8-GPU shard size on one GPU
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for off in 0 1 0 1; do
  echo "== LIFE_B200_NO_TILE_ROUND=$off"
  LIFE_B200_NO_TILE_ROUND=$off timeout 600 python tools/bin_check.py --c2 2>&1 | grep -E "^C1|^C2|^tiny|^nt=150|bad"
  for cfg in c2x8 c2; do
    LIFE_B200_NO_TILE_ROUND=$off timeout 600 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu --no-e2e 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value'],1), 'it/s dsc', round(d['spmv']['dsc_ms'],4), 'wc', round(d['spmv']['wc_ms'],4))"
  done
done
