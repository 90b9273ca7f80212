#!/bin/bash
# A/B of the decode CTA sizes (LA2_DEC1_THREADS / LA2_DECT_THREADS build variants):
# VARIANTS="t64 ..." -> paper_2401_04658_b200/libla2_<v>.so against the committed build
mkdir -p gpurun_out; O=gpurun_out/ab_decode_cta.txt; : > $O
for i in 1 2; do for v in base ${VARIANTS:-d128}; do
  if [ $v = base ]; then L=$PWD/paper_2401_04658_b200/libla2.so; else L=$PWD/paper_2401_04658_b200/libla2_$v.so; fi
  echo "--- $v" >> $O
  LA2_LIB=$L python tools/decode_multi.py 64 > /tmp/dm.txt 2>&1; grep -E "single|T=  1:|T=  4:|T=  8:|T= 64:" /tmp/dm.txt >> $O
  LA2_LIB=$L python tools/decode_multi.py 256 > /tmp/dm.txt 2>&1; grep -E "single|T=  1:|T=  4:|T=  8:|T= 16:|T= 64:" /tmp/dm.txt >> $O
done; done
cat $O
