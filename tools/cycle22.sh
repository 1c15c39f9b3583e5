#!/bin/bash
# L1 prefetch of each slice's edge records (main build) vs without (variants/libshift.so).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/c22_pytest.log
O=gpurun_out/c22_ab.jsonl; : > $O
V=$PWD/paper_2402_08296_b200/variants
for i in 1 2 3; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"prefetch",/' >> $O
  DDMGNN_B200_LIB=$V/libshift.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"shift",/' >> $O
done
SUBDOMAIN_SIZE=500 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"prefetch",/' >> $O
SUBDOMAIN_SIZE=500 DDMGNN_B200_LIB=$V/libshift.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"shift",/' >> $O
cat gpurun_out/c22_pytest.log $O
