#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/c13_cl2.jsonl; : > $O
L=$PWD/paper_2402_08296_b200/variants/libcl2.so
for NS in 2000 5000; do
  SUBDOMAIN_SIZE=$NS timeout 300 python tools/time_apply.py 2>&1 | tail -1 >> $O
  SUBDOMAIN_SIZE=$NS DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"cl2",/' >> $O
done
timeout 300 python tools/time_apply.py 2>&1 | tail -1 >> $O
DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"cl2",/' >> $O
DDMGNN_CAP0=0 timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"cap0",/' >> $O
DDMGNN_CAP0=0 DDMGNN_B200_LIB=$L timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"cl2 cap0",/' >> $O
cat $O
