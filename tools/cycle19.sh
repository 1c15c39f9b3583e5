#!/bin/bash
# Edge-loop shift form (GNN_EDGE_SHIFT=1, main build) vs the previous form (variants/libold.so):
# GPU parity tests on the main build, then alternating apply timings at config C and E(N_s=500).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/c19_pytest.log
O=gpurun_out/c19_ab.jsonl; : > $O
L=$PWD/paper_2402_08296_b200/variants/libold.so
for i in 1 2 3; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"shift",/' >> $O
  DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"old",/' >> $O
done
SUBDOMAIN_SIZE=500 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"shift",/' >> $O
SUBDOMAIN_SIZE=500 DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"old",/' >> $O
cat gpurun_out/c19_pytest.log $O
