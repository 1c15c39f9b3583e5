#!/bin/bash
# Profiling pass of one round (run under gpurun, 1 GPU):
#   * launch list (per-launch device time, cold & serialised) of 3 applies + 3 SpMVs
#   * one `ncu --set full` capture of gnn_kernel, gnn_cluster_kernel and the SpMV
# Outputs land in gpurun_out/; tools/summarise_profiles.py turns them into profiles/.
R=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python tools/profile_apply.py > gpurun_out/${R}_launches.log 2>&1
for K in gnn_kernel gnn_cluster_kernel spmv_kernel; do
  ncu --set full --clock-control none --import-source on -k ${K} -s 1 -c 1 \
      -o gpurun_out/${R}_${K} python tools/profile_apply.py > gpurun_out/${R}_${K}.log 2>&1
done
ls -la gpurun_out/${R}_*
