#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/exp3.jsonl
: > $O
for v in 1 3; do
  L=$PWD/paper_2402_08296_b200/variants/libcl$v.so
  DDMGNN_B200_LIB=$L python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"v\":\"cl$v\",/" >> $O
  DDMGNN_B200_LIB=$L DDMGNN_CAP0=0 DDMGNN_CLUSTER_2CTA=1 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"v\":\"cl$v cap0 2cta\",/" >> $O
  DDMGNN_B200_LIB=$L DDMGNN_CAP0=0 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"v\":\"cl$v cap0\",/" >> $O
done
cat $O
