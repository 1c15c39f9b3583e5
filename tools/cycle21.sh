#!/bin/bash
# ncu --set full of gnn_kernel (shift-form edge loop) at config C.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gnn_kernel -s 1 -c 1 \
    -o gpurun_out/r02_gnn_shift python tools/profile_apply.py --applies 2 > gpurun_out/c21_ncu.log 2>&1
tail -2 gpurun_out/c21_ncu.log; ls -la gpurun_out/
