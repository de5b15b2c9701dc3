#!/bin/bash
# round-2 GPU check: full -m gpu suite (no -x: every failure listed), then
# the reference arm at full C2 and the default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
if [ "${WITH_REF:-0}" = 1 ]; then
  t0=$(date +%s)
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "reference arm wall: $(( $(date +%s) - t0 )) s" >> gpurun_out/bench_ref.err
  tail -c 2000 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
