#!/bin/bash
# round-2 cycle 4: full GPU tests, default bench, config D record (10M DOFs, 1 GPU),
# ncu capture of the GNN kernel.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/c4_pytest.log 2>&1
tail -8 gpurun_out/c4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c4_smoke.log 2>&1; tail -1 gpurun_out/c4_smoke.log
timeout 1200 python bench.py > gpurun_out/c4_bench.json 2> gpurun_out/c4_bench.err; tail -c 300 gpurun_out/c4_bench.json
timeout 1200 python bench.py --target-nodes 10000000 --no-cpu --steps 10 --warmup 3 > gpurun_out/c4_configD.json 2> gpurun_out/c4_configD.err
tail -c 600 gpurun_out/c4_configD.json; tail -3 gpurun_out/c4_configD.err
ncu --set full --clock-control none --import-source on -k regex:gnn_kernel -s 1 -c 1 \
    -o gpurun_out/r02_gnn_h0 python tools/profile_apply.py --applies 2 > gpurun_out/r02_gnn_h0_ncu.log 2>&1
tail -1 gpurun_out/r02_gnn_h0_ncu.log
