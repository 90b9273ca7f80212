mkdir -p gpurun_out
python tools/fbench.py 8,16,65536,64 > gpurun_out/e_fb1.txt 2>&1
python bench.py --no-sweep --no-e2e --no-cpu > gpurun_out/e_bench.json 2>&1
python tools/fbench.py 8,16,65536,64 > gpurun_out/e_fb2.txt 2>&1
python -m pytest tests/test_gpu_parity.py -q -k decode > gpurun_out/e_dec.txt 2>&1
python bench.py --workload c4 --steps 10 > gpurun_out/e_c4.json 2>&1
