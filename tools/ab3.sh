#!/bin/bash
# A/B/C of alternative builds on one box (development): base, h0, h4096
mkdir -p gpurun_out
S=${AB_SHAPES:-"8,16,65536,64 32,16,16384,128 4,20,16384,128"}
: > gpurun_out/ab3.txt
for i in 1 2; do
  for v in base h0 h4096; do
    echo "--- $v" >> gpurun_out/ab3.txt
    LA2_LIB=$PWD/paper_2401_04658_b200/libla2_$v.so timeout 120 python tools/fbench.py $S >> gpurun_out/ab3.txt 2>&1
  done
done
