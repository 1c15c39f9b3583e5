#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/c17_pf.jsonl; : > $O
L=$PWD/paper_2402_08296_b200/variants/libpf.so
for i in 1 2; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 >> $O
  DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"q_prefetch",/' >> $O
done
SUBDOMAIN_SIZE=500 timeout 300 python tools/time_apply.py 2>&1 | tail -1 >> $O
SUBDOMAIN_SIZE=500 DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"q_prefetch",/' >> $O
cat $O
