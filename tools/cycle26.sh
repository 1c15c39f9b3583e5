#!/bin/bash
# Round-2 final profiles of the dataflow kernel: launch list of a short bench run (the
# bench's own timed applies, cold and serialised under ncu), ncu --set full of gnn_kernel,
# and the PCG-iteration launch list with DRAM bytes.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02f_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-pcg \
    > gpurun_out/c26_bench_ncu.log 2>&1
tail -c 200 gpurun_out/c26_bench_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gnn_kernel -s 1 -c 1 \
    -o gpurun_out/r02f_gnn python tools/profile_apply.py --applies 2 > gpurun_out/c26_gnn_ncu.log 2>&1
tail -2 gpurun_out/c26_gnn_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02f_pcg_launches.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c26_pcg.log 2>&1
tail -1 gpurun_out/c26_pcg.log
ls -la gpurun_out
