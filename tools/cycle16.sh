#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_final.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c16_launches.log 2>&1
tail -1 gpurun_out/c16_launches.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gnn_kernel -s 1 -c 1 \
    -o gpurun_out/r02_gnn_final python tools/profile_apply.py --applies 2 > gpurun_out/c16_gnn_ncu.log 2>&1
tail -1 gpurun_out/c16_gnn_ncu.log
timeout 1200 python bench.py > gpurun_out/c16_bench.json 2> gpurun_out/c16_bench.err; tail -c 300 gpurun_out/c16_bench.json
