#!/bin/bash
# A/B: d=128 one V~ buffer + double-buffered O staging vs two V~ buffers + one O staging (development)
mkdir -p gpurun_out; : > gpurun_out/ab_kts.txt
S="32,16,16384,128 4,20,16384,128"
for i in 1 2 3; do for v in base kts1; do
  echo "--- $v" >> gpurun_out/ab_kts.txt
  LA2_LIB=$PWD/paper_2401_04658_b200/libla2_$v.so timeout 120 python tools/fbench.py $S >> gpurun_out/ab_kts.txt 2>&1
done; done
LA2_LIB=$PWD/paper_2401_04658_b200/libla2_kts1.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "random_shapes or persistent or quad or d128 or 128" > gpurun_out/t_kts.txt 2>&1
