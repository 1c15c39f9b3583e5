#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/c6_e2e.jsonl; : > $O
for i in 1 2; do
  python tools/e2e_ab.py 2>&1 | tail -1 >> $O
  DDMGNN_STAGED_INPUT=0 python tools/e2e_ab.py 2>&1 | tail -1 >> $O
done
cat $O
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=3 > gpurun_out/c6_pytest.log 2>&1
tail -5 gpurun_out/c6_pytest.log
