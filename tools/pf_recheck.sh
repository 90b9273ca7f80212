mkdir -p gpurun_out; : > gpurun_out/pf.txt
S="32,16,16384,128 4,20,16384,128"
for i in 1 2; do for pf in 0 1 2 4; do for h in 0 2; do echo "--- pf=$pf hint=$h" >> gpurun_out/pf.txt; LA2_PF=$pf LA2_HINT=$h timeout 100 python tools/fbench.py $S >> gpurun_out/pf.txt 2>&1; done; done; done
