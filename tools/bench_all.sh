#!/bin/bash
# All bench workloads (BASELINE configs) -> gpurun_out/bench_<w>.json
mkdir -p gpurun_out
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 10 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
