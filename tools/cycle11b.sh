#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/c11b_e2e.jsonl; : > $O
timeout 300 python tools/e2e_ab.py 2>&1 | tail -1 >> $O
DDMGNN_STAGED_INPUT=0 timeout 300 python tools/e2e_ab.py 2>&1 | tail -1 >> $O
timeout 300 python tools/e2e_ab.py 2>&1 | tail -1 >> $O
cat $O
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/c11b_pytest.log 2>&1; tail -3 gpurun_out/c11b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/c11b_bench.json 2> gpurun_out/c11b_bench.err; tail -c 200 gpurun_out/c11b_bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gnn_cluster_kernel -s 1 -c 1 \
    -o gpurun_out/r02_cluster_ns2000 python tools/profile_apply.py --subdomain-size 2000 --applies 2 > gpurun_out/c12_ncu.log 2>&1
tail -1 gpurun_out/c12_ncu.log
