#!/bin/bash
# d=128 F kernel: DRAM bytes and time vs L2 prefetch distance / clusters (development).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for pf in 0 1 2 3 6; do
  LA2_PF=$pf ncu --metrics $M --clock-control none --csv -k regex:la2_tc_kernel -c 4 --log-file gpurun_out/pf_$pf.csv \
    python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 1 > /dev/null 2>&1
  LA2_PF=$pf python tools/fbench.py 32,16,16384,128 4,20,16384,128 > gpurun_out/pf_time_$pf.txt 2>&1
done
LA2_NO_CLUSTER=1 LA2_PF=0 ncu --metrics $M --clock-control none --csv -k regex:la2_tc_kernel -c 4 --log-file gpurun_out/pf_nocl.csv \
    python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 1 > /dev/null 2>&1
