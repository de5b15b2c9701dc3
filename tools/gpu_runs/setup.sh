#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/setup_breakdown.py > gpurun_out/setup.log 2>&1
