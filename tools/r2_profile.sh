#!/bin/bash
# Round-2 evidence: default bench line, ncu launch list of the bench command, ncu --set full
# of every tcgen05 launch of one C2-shape step (N=16K) -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --soak-s 0.01 --no-sweep --no-e2e --no-cpu --no-parity \
    > gpurun_out/launches_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 2 -c 2 \
    -o gpurun_out/full_d64 -f python tools/prof_step.py --seq-len 16384 --steps 2 > gpurun_out/full_d64.log 2>&1
echo done > gpurun_out/r2_profile.done
