#!/bin/bash
# A/B on one box, alternating: committed baseline lib vs the working tree lib (development).
mkdir -p gpurun_out
S=${AB_SHAPES:-"8,16,65536,64 32,16,16384,128 4,20,16384,128"}
: > gpurun_out/ab.txt
for i in 1 2 3; do
  echo "--- base" >> gpurun_out/ab.txt
  LA2_LIB=$PWD/paper_2401_04658_b200/libla2_base.so timeout 120 python tools/fbench.py $S >> gpurun_out/ab.txt 2>&1
  echo "--- new" >> gpurun_out/ab.txt
  timeout 120 python tools/fbench.py $S >> gpurun_out/ab.txt 2>&1
done
