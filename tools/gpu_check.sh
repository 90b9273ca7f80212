#!/bin/bash
# First-pass GPU validation: layouts, smoke, parity, short bench. Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_selftest.py -q -x -rA > gpurun_out/selftest.log 2>&1
echo "selftest rc=$?" >> gpurun_out/summary.txt
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
rc=$?
echo "smoke rc=$rc" >> gpurun_out/summary.txt
if [ $rc -eq 0 ]; then
  timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rA -s > gpurun_out/parity.log 2>&1
  echo "parity rc=$?" >> gpurun_out/summary.txt
  timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/summary.txt
else
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -rA -s -k "simt or tila or decode or fp32" > gpurun_out/parity_simt.log 2>&1
  echo "parity(simt) rc=$?" >> gpurun_out/summary.txt
fi
