#!/bin/bash
# Re-entry check of the round-2 tree on a fresh box: GPU tests, smoke, default bench, apply timing.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/c18_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c18_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c18_bench.json 2> gpurun_out/c18_bench.err
timeout 300 python tools/time_apply.py > gpurun_out/c18_time.jsonl 2>&1
cat gpurun_out/c18_pytest.log gpurun_out/c18_smoke.log; tail -2 gpurun_out/c18_time.jsonl
python -c "import json;d=json.load(open('gpurun_out/c18_bench.json'));print({k:d[k] for k in ('value','ms_per_step','e2e','clocks')});print(d['roofline'])"
