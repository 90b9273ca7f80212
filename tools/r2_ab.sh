#!/bin/bash
# A/B of several library builds on one box: LIBS="name:path ..." SHAPES="B,H,N,d ..."
mkdir -p gpurun_out
O=${AB_OUT:-gpurun_out/ab.txt}
: > $O
for i in 1 2; do
  for spec in $LIBS; do
    n=${spec%%:*}; l=${spec#*:}
    echo "--- $n" >> $O
    LA2_LIB=$PWD/$l timeout 300 python tools/stepbench.py $SHAPES >> $O 2>&1
  done
done
