#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_step.py --seq-len 65536 --steps 2 > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 4 -c 4 \
    -o gpurun_out/prof_tc python tools/prof_step.py --seq-len 16384 --steps 2 > gpurun_out/prof.log 2>&1
echo "rc=$?" >> gpurun_out/prof.log
