#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_sus.txt
for i in 1 2; do
  for v in base new; do
    echo "--- $v" >> gpurun_out/ab_sus.txt
    LA2_LIB=$PWD/paper_2401_04658_b200/libla2_$v.so timeout 200 python tools/sustained.py >> gpurun_out/ab_sus.txt 2>&1
  done
done
