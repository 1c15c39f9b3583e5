#!/bin/bash
# Dataflow race/equality test, 768-thread variant A/B, default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dataflow.py -x -q 2>&1 | tail -3 > gpurun_out/c25_pytest.log
O=gpurun_out/c25_ab.jsonl; : > $O
V=$PWD/paper_2402_08296_b200/variants
for i in 1 2; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"t896",/' >> $O
  DDMGNN_B200_LIB=$V/libt768.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"t768",/' >> $O
done
timeout 900 python bench.py > gpurun_out/c25_bench.json 2> gpurun_out/c25_bench.err
cat gpurun_out/c25_pytest.log $O
python -c "import json;d=json.load(open('gpurun_out/c25_bench.json'));print({k:d[k] for k in ('value','ms_per_step','e2e','clocks')});print(d['roofline']['frac'],d['roofline']['frac_executed'],d['roofline']['gnn_ms']);print(d['pcg']);print(d['pcg_flexible'])"
