#!/bin/bash
# Final round-2 check: all GPU tests, smoke, default bench, N_s=500/overlap-1 A/B, config E sweep.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/c30_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c30_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c30_bench.json 2> gpurun_out/c30_bench.err
O=gpurun_out/c30_ab.jsonl; : > $O
for DF in 1 0; do
  OVERLAP=1 SUBDOMAIN_SIZE=500 DDMGNN_DATAFLOW=$DF timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"overlap\":1,\"df\":$DF,/" >> $O
  DDMGNN_DATAFLOW=$DF timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"df\":$DF,/" >> $O
done
timeout 1800 python tools/sweep.py --min-nodes 1000000 > gpurun_out/c30_sweep.jsonl 2> gpurun_out/c30_sweep.err
cat gpurun_out/c30_pytest.log gpurun_out/c30_smoke.log $O; wc -l gpurun_out/c30_sweep.jsonl
python -c "import json;d=json.load(open('gpurun_out/c30_bench.json'));print({k:d[k] for k in ('value','ms_per_step','e2e','clocks','gpu_launches')});print(d['roofline']['frac'],d['roofline']['frac_executed'],d['roofline']['gnn_ms']);print(d['pcg']['seconds'],d['pcg']['iterations'],d['pcg_flexible']['seconds'],d['pcg_flexible']['iterations'])"
