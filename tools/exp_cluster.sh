#!/bin/bash
# Round-2 experiment: all subdomains of config C on 2-CTA clusters (2 CTAs / SM),
# with and without the local-row fast path of ClusterRows; plus one ncu capture.
mkdir -p gpurun_out
O=gpurun_out/exp2.jsonl
: > $O
python tools/time_apply.py >> $O
DDMGNN_CAP0=0 DDMGNN_CLUSTER_2CTA=1 python tools/time_apply.py | sed 's/^{/{"v":"cap0 2cta",/' >> $O
DDMGNN_CAP0=0 python tools/time_apply.py | sed 's/^{/{"v":"cap0",/' >> $O
for v in 1 3; do
  DDMGNN_B200_LIB=$PWD/paper_2402_08296_b200/variants/libcl$v.so python tools/time_apply.py | sed "s/^{/{\"v\":\"cl$v\",/" >> $O
  DDMGNN_B200_LIB=$PWD/paper_2402_08296_b200/variants/libcl$v.so DDMGNN_CAP0=0 DDMGNN_CLUSTER_2CTA=1 python tools/time_apply.py | sed "s/^{/{\"v\":\"cl$v cap0 2cta\",/" >> $O
  DDMGNN_B200_LIB=$PWD/paper_2402_08296_b200/variants/libcl$v.so DDMGNN_CAP0=0 python tools/time_apply.py | sed "s/^{/{\"v\":\"cl$v cap0\",/" >> $O
done
cat $O
ncu --set full --clock-control none --import-source on -k regex:gnn_kernel -s 1 -c 1 \
    -o gpurun_out/r02_gnn python tools/profile_apply.py --applies 2 > gpurun_out/r02_gnn_ncu.log 2>&1
tail -3 gpurun_out/r02_gnn_ncu.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches.csv python tools/profile_pcg.py --iters 6 > gpurun_out/r02_pcg_launches.log 2>&1
tail -2 gpurun_out/r02_pcg_launches.log
