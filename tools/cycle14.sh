#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/c14_e2e.jsonl; : > $O
for i in 1 2; do
timeout 300 python tools/e2e_ab.py 2>&1 | tail -1 | sed 's/^{/{"zero_copy_out":1,/' >> $O
DDMGNN_ZERO_COPY_OUT=0 timeout 300 python tools/e2e_ab.py 2>&1 | tail -1 | sed 's/^{/{"zero_copy_out":0,/' >> $O
done
cat $O
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/c14_pytest.log 2>&1; tail -3 gpurun_out/c14_pytest.log
