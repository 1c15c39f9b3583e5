#!/bin/bash
# Last check of the committed tree: all GPU tests, smoke, default bench.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/c33_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c33_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c33_bench.json 2> gpurun_out/c33_bench.err
cat gpurun_out/c33_pytest.log gpurun_out/c33_smoke.log
python -c "import json;d=json.load(open('gpurun_out/c33_bench.json'));print({k:d[k] for k in ('value','ms_per_step','e2e','clocks','gpu_launches')});print(d['roofline']['frac'],d['roofline']['frac_executed'],d['roofline']['gnn_ms'],d['roofline']['traffic']);print(d['pcg']['seconds'],d['pcg']['iterations'],d['pcg_flexible']['seconds'],d['pcg_flexible']['iterations'])"
