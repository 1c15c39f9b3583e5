#!/bin/bash
# Dataflow knobs: phase-A items as slice pairs (main) or single slices (s*), poll sleep 20 or 100 ns.
mkdir -p gpurun_out
O=gpurun_out/c27_ab.jsonl; : > $O
V=$PWD/paper_2402_08296_b200/variants
for i in 1 2; do
  timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"p20",/' >> $O
  for n in s20 p100 s100; do
    DDMGNN_B200_LIB=$V/lib$n.so timeout 300 python tools/time_apply.py 2>&1 | tail -1 | sed "s/^{/{\"v\":\"$n\",/" >> $O
  done
done
cat $O
