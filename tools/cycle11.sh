#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/c11_e2e.jsonl; : > $O
python tools/e2e_ab.py 2>&1 | tail -1 >> $O
DDMGNN_STAGED_INPUT=0 python tools/e2e_ab.py 2>&1 | tail -1 >> $O
python tools/e2e_ab.py 2>&1 | tail -1 >> $O
cat $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_c11.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c11_launches.log 2>&1
tail -1 gpurun_out/c11_launches.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/c11_pytest.log 2>&1; tail -3 gpurun_out/c11_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/c11_bench.json 2> gpurun_out/c11_bench.err; tail -c 200 gpurun_out/c11_bench.json
