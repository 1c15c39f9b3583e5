#!/bin/bash
# Candidate: dataflow polls with exponential back-off (16..256 ns) and the dataflow
# schedule also in two-CTA mode (variants/libcand.so) vs the committed build.
mkdir -p gpurun_out
V=$PWD/paper_2402_08296_b200/variants
DDMGNN_B200_LIB=$V/libcand.so timeout 900 python -m pytest tests/test_gpu_dataflow.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2 > gpurun_out/c31_pytest.log
O=gpurun_out/c31_ab.jsonl; : > $O
for i in 1 2; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"main",/' >> $O
  DDMGNN_B200_LIB=$V/libcand.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"cand",/' >> $O
done
for OV in 1 2 3; do
  OVERLAP=$OV SUBDOMAIN_SIZE=500 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"v\":\"main\",\"overlap\":$OV,/" >> $O
  OVERLAP=$OV SUBDOMAIN_SIZE=500 DDMGNN_B200_LIB=$V/libcand.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"v\":\"cand\",\"overlap\":$OV,/" >> $O
done
cat gpurun_out/c31_pytest.log $O
