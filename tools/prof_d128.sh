#!/bin/bash
# d=128 launch lists (C3, C4 shapes) + one full ncu capture of the d=128 F kernel.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 2 > gpurun_out/l3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python tools/prof_step.py --seq-len 16384 --batch 4 --heads 20 --dim 128 --steps 2 > gpurun_out/l4.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python tools/prof_step.py --seq-len 65536 --batch 8 --dim 64 --steps 2 > gpurun_out/l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 4 -c 1 \
    -o gpurun_out/prof_d128 python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 2 > gpurun_out/prof.log 2>&1
echo "rc=$?" >> gpurun_out/prof.log
