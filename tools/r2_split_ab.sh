#!/bin/bash
# Shared-recurrence backward pair/triple (LA2_SPLIT_STATE): quick parity first (short
# timeout: a hang must not hold the GPU), then the full GPU suite, then an A/B of the
# step against the previous build (libla2_base.so) on the same box.
mkdir -p gpurun_out
O=gpurun_out/r2_split
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "backward_with_carried or tc_forward_backward or stored_states" > $O.quick.log 2>&1
echo "quick rc=$?" >> $O.quick.log
if grep -q "quick rc=0" $O.quick.log; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O.gputest.log 2>&1; echo "rc=$?" >> $O.gputest.log
  S="8,16,65536,64 8,16,16384,64 8,16,4096,64 8,16,1024,64"
  : > $O.ab.txt
  for i in 1 2; do
    echo "--- base" >> $O.ab.txt
    LA2_LIB=$PWD/paper_2401_04658_b200/libla2_base.so timeout 300 python tools/stepbench.py $S >> $O.ab.txt 2>&1
    echo "--- new" >> $O.ab.txt
    timeout 300 python tools/stepbench.py $S >> $O.ab.txt 2>&1
  done
fi
