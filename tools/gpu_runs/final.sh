#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/qb.json 2> gpurun_out/qb.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --layout fma > gpurun_out/qb_fma.json 2>> gpurun_out/qb.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
