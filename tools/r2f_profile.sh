#!/bin/bash
# Round-2 (final kernels) evidence -> gpurun_out/r2f_*: ncu launch list of the default bench
# command (C2), ncu --set full of one fwd+bwd step at the C2 shape (N=16K: forward storing
# the states + dQ/dK/dV triple) and at d=128 (B=8 H=16 N=16K: forward F, dQ F, dK F, dV F).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/r2f_launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --soak-s 0.01 --no-sweep --no-e2e --no-cpu --no-parity \
    > gpurun_out/r2f_launches_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 2 -c 2 \
    -o gpurun_out/r2f_full_d64 -f python tools/prof_step.py --seq-len 16384 --steps 2 > gpurun_out/r2f_full_d64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 4 -c 4 \
    -o gpurun_out/r2f_full_d128 -f python tools/prof_step.py --seq-len 16384 --dim 128 --steps 2 > gpurun_out/r2f_full_d128.log 2>&1
echo done > gpurun_out/r2f_profile.done
