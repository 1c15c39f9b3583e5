#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_c10.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c10_launches.log 2>&1
tail -1 gpurun_out/c10_launches.log
python tools/time_pcg.py 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/c10_pytest.log 2>&1; tail -3 gpurun_out/c10_pytest.log
timeout 1200 python bench.py --no-cpu > gpurun_out/c10_bench.json 2> gpurun_out/c10_bench.err; tail -c 200 gpurun_out/c10_bench.json
