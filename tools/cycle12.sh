#!/bin/bash
# cluster-path profile at BASELINE config E N_s = 2000 (every subdomain on 2-CTA clusters)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gnn_cluster_kernel -s 1 -c 1 \
    -o gpurun_out/r02_cluster_ns2000 python tools/profile_apply.py --subdomain-size 2000 --applies 2 > gpurun_out/c12_ncu.log 2>&1
tail -2 gpurun_out/c12_ncu.log
