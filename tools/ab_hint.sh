#!/bin/bash
# A/B of mbarrier try_wait suspend hints (development)
mkdir -p gpurun_out; : > gpurun_out/ab_hint.txt
S="8,16,65536,64 32,16,16384,128"
for i in 1 2; do for v in base h0 h100 h1000; do
  echo "--- $v" >> gpurun_out/ab_hint.txt
  LA2_LIB=$PWD/paper_2401_04658_b200/libla2_$v.so timeout 120 python tools/fbench.py $S >> gpurun_out/ab_hint.txt 2>&1
done; done
