#!/bin/bash
# C5 sweep on the binned products (lognormal 1M..1B, Zipf up to 256M) + the generator test
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_skew.py -q -p no:cacheprovider -k device_generator 2>&1 | tail -2
timeout 900 python tools/sweep_c5.py --nnz 1e6,4e6,16e6,64e6,256e6 --skew lognormal > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
timeout 900 python tools/sweep_c5.py --nnz 16e6,64e6,256e6 --skew zipf >> gpurun_out/sweep_c5.jsonl 2>> gpurun_out/sweep_c5.err
timeout 900 python tools/sweep_c5.py --nnz 1e9 --skew lognormal --reps 10 >> gpurun_out/sweep_c5.jsonl 2>> gpurun_out/sweep_c5.err
tail -3 gpurun_out/sweep_c5.err
python - <<'PY'
import json
for l in open("gpurun_out/sweep_c5.jsonl"):
    d = json.loads(l)
    p = d.get("parity", {})
    print(d["skew"], d["nnz"], d["op"], d["kernels"], d["ms"], d["gbs"], d["frac"], d["max_fascicle_len"], p.get("dsc_rel_l2"), p.get("wc_rel_l2"))
PY
