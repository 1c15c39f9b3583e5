#!/bin/bash
# Dataflow layer schedule of the CTA path (default) vs two barriers per layer (DDMGNN_DATAFLOW=0).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/c23_pytest.log
O=gpurun_out/c23_ab.jsonl; : > $O
for i in 1 2 3; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"dataflow",/' >> $O
  DDMGNN_DATAFLOW=0 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"barriers",/' >> $O
done
for NS in 500 2000; do
SUBDOMAIN_SIZE=$NS timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"dataflow",/' >> $O
SUBDOMAIN_SIZE=$NS DDMGNN_DATAFLOW=0 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"barriers",/' >> $O
done
cat gpurun_out/c23_pytest.log $O
