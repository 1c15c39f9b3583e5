#!/bin/bash
# update / p-update kernels with two 16-byte pairs per step: PCG tests and the PCG-iteration launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_north_star.py -x -q -k "pcg or cg or fcg" 2>&1 | tail -2 > gpurun_out/c32_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02g_pcg_launches.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c32_pcg.log 2>&1
timeout 300 python tools/time_pcg.py > gpurun_out/c32_time_pcg.txt 2>&1
cat gpurun_out/c32_pytest.log; tail -3 gpurun_out/c32_time_pcg.txt
