#!/bin/bash
# Cluster-path dataflow + the N_s=500/overlap-1 regression: dataflow vs barriers, one vs two CTAs per SM.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dataflow.py -x -q 2>&1 | tail -3 > gpurun_out/c29_pytest.log
O=gpurun_out/c29_ab.jsonl; : > $O
for KB in 5 10; do
for DF in 1 0; do for TC in 1 0; do
  KBAR=$KB OVERLAP=1 SUBDOMAIN_SIZE=500 DDMGNN_DATAFLOW=$DF DDMGNN_TWO_CTA=$TC timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"kbar\":$KB,\"df\":$DF,\"two_cta\":$TC,/" >> $O
done; done; done
for NS in 2000 5000; do for DF in 1 0; do
  SUBDOMAIN_SIZE=$NS DDMGNN_DATAFLOW=$DF timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"df\":$DF,/" >> $O
done; done
for DF in 1 0; do
  DDMGNN_DATAFLOW=$DF timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"df\":$DF,/" >> $O
done
cat gpurun_out/c29_pytest.log $O
