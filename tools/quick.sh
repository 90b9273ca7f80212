#!/bin/bash
# Quick GPU loop: parity tests (optionally filtered) + kernel timings. Logs -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/q_summary.txt
timeout 300 python tools/fbench.py ${FB_SHAPES:-8,16,65536,64 32,16,16384,128 4,20,16384,128 1,16,131072,128} > gpurun_out/q_fbench.txt 2>&1
echo "fbench rc=$?" >> gpurun_out/q_summary.txt
