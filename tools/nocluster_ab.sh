#!/bin/bash
# A/B: 2-CTA multicast clusters vs independent CTAs (L2 sharing) at d=128 (development)
mkdir -p gpurun_out; : > gpurun_out/nocl.txt
S="32,16,16384,128 4,20,16384,128 8,16,65536,64"
for i in 1 2; do
  echo "--- cluster" >> gpurun_out/nocl.txt; timeout 120 python tools/fbench.py $S >> gpurun_out/nocl.txt 2>&1
  echo "--- nocluster" >> gpurun_out/nocl.txt; LA2_NO_CLUSTER=1 timeout 120 python tools/fbench.py $S >> gpurun_out/nocl.txt 2>&1
done
