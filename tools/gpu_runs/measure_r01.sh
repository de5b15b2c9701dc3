#!/bin/bash
# round-1 measurement set: bench (our arm + reference arm), ncu launch list, ncu full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(dsc_tc|wc_tc)" -s 2 -c 2 -o gpurun_out/ws_full -f python tools/prof_spmv.py --reps 3 > gpurun_out/ncu_full.log 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
