#!/bin/bash
# A/B: LSU L2 prefetch from the producer warp's idle lanes (LA2_PF < 0) at d=128 (development)
mkdir -p gpurun_out; : > gpurun_out/ab_lsupf.txt
S="32,16,16384,128 4,20,16384,128"
for i in 1 2; do
  for pf in 0 -1 -2 -3; do
    echo "--- pf=$pf" >> gpurun_out/ab_lsupf.txt
    LA2_PF=$pf timeout 120 python tools/fbench.py $S >> gpurun_out/ab_lsupf.txt 2>&1
  done
done
LA2_PF=-2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "random_shapes or persistent or views or long_sequence" > gpurun_out/t_lsupf.txt 2>&1
