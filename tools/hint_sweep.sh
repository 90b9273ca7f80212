#!/bin/bash
# d=128 F kernel: DRAM bytes and time vs L2 prefetch distance and cache-policy hints (development).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in "3 0" "3 3" "3 7" "2 3" "4 3" "6 3" "3 2" "1 3"; do
  set -- $cfg
  LA2_PF=$1 LA2_HINT=$2 ncu --metrics $M --clock-control none --csv -k regex:la2_tc_kernel -c 2 --log-file gpurun_out/h_$1_$2.csv \
    python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 1 > /dev/null 2>&1
  echo "PF=$1 HINT=$2" >> gpurun_out/h_time.txt
  LA2_PF=$1 LA2_HINT=$2 python tools/fbench.py 32,16,16384,128 >> gpurun_out/h_time.txt 2>&1
done
LA2_HINT=7 python tools/fbench.py 8,16,65536,64 >> gpurun_out/h_time.txt 2>&1
python tools/fbench.py 8,16,65536,64 >> gpurun_out/h_time.txt 2>&1
