#!/bin/bash
mkdir -p gpurun_out
S="8,16,65536,64 32,16,16384,128 4,20,16384,128"
python tools/fbench.py $S > gpurun_out/ab_new.txt 2>&1
python tools/trace.py 16384 64 > gpurun_out/trace64.txt 2>&1
