#!/bin/bash
# Full bench + ncu evidence for profiles/. Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_step.py --seq-len 65536 --steps 2 > gpurun_out/launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/summary.txt
ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 4 -c 4 \
    -o gpurun_out/prof_tc python tools/prof_step.py --seq-len 16384 --steps 2 > gpurun_out/prof.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/summary.txt
