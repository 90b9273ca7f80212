#!/bin/bash
# Round evidence for profiles/: all bench workloads, ncu launch lists (time + DRAM bytes)
# of one fwd+bwd step at the C2 and C3 shapes, and ncu --set full of every tcgen05
# launch of one step (C2 shape at N=16K, d=128 shape at B=8 N=16K). Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
bash tools/bench_all.sh
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python tools/prof_step.py --seq-len 65536 --steps 2 > gpurun_out/launches_c2.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 2 > gpurun_out/launches_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 3 -c 3 \
    -o gpurun_out/full_d64 python tools/prof_step.py --seq-len 16384 --steps 2 > gpurun_out/full_d64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:la2_tc_kernel -s 3 -c 3 \
    -o gpurun_out/full_d128 python tools/prof_step.py --seq-len 16384 --batch 8 --dim 128 --steps 2 > gpurun_out/full_d128.log 2>&1
echo done > gpurun_out/round_profile.done
