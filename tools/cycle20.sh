#!/bin/bash
# Edge loop: shift form + two half passes with two edges in flight (main build) vs
# shift form alone (variants/libshift.so) vs the previous form (variants/libold.so).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/c20_pytest.log
O=gpurun_out/c20_ab.jsonl; : > $O
V=$PWD/paper_2402_08296_b200/variants
for i in 1 2 3; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"halves",/' >> $O
  DDMGNN_B200_LIB=$V/libshift.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"shift",/' >> $O
  DDMGNN_B200_LIB=$V/libold.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"old",/' >> $O
done
SUBDOMAIN_SIZE=500 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"halves",/' >> $O
SUBDOMAIN_SIZE=500 DDMGNN_B200_LIB=$V/libshift.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"shift",/' >> $O
cat gpurun_out/c20_pytest.log $O
