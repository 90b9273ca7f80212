ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__cluster_dim_x --clock-control none --csv --log-file gpurun_out/launches_c3q.csv \
    python tools/prof_step.py --seq-len 16384 --batch 32 --dim 128 --steps 1 > /dev/null 2>&1
