#!/bin/bash
# round-2 cycle 8: grid-stride SpMV (fewer reduction partials) — launch list, ncu
# --set full of the per-iteration vector kernels, GPU tests, bench line.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_c8.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c8_launches.log 2>&1
tail -1 gpurun_out/c8_launches.log
ncu --set full --clock-control none --import-source on -k regex:"spmv_kernel|update_kernel|prolong_kernel|pupdate_kernel|coarse_gemv" -s 8 -c 5 \
    -o gpurun_out/r02_vec_full python tools/profile_pcg.py --iters 4 > gpurun_out/c8_vec_ncu.log 2>&1
tail -1 gpurun_out/c8_vec_ncu.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/c8_pytest.log 2>&1; tail -3 gpurun_out/c8_pytest.log
timeout 1200 python bench.py --no-cpu > gpurun_out/c8_bench.json 2> gpurun_out/c8_bench.err; tail -c 200 gpurun_out/c8_bench.json
