#!/bin/bash
# A/B: ring depth of the state-only passes (development)
mkdir -p gpurun_out; : > gpurun_out/ab_so.txt
for i in 1 2; do for v in base so3 so4; do
  echo "--- $v" >> gpurun_out/ab_so.txt
  LA2_LIB=$PWD/paper_2401_04658_b200/libla2_$v.so timeout 200 python tools/so_bench.py >> gpurun_out/ab_so.txt 2>&1
done; done
