#!/bin/bash
# round-2 cycle 9: edge-pair GNN variant A/B, one-pair-per-thread vector kernels
# (launch list), GPU tests.
mkdir -p gpurun_out
O=gpurun_out/c9_ab.jsonl; : > $O
python tools/time_apply.py 2>&1 | tail -1 >> $O
DDMGNN_B200_LIB=$PWD/paper_2402_08296_b200/variants/libpair.so python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"edge_pair",/' >> $O
python tools/time_apply.py 2>&1 | tail -1 >> $O
DDMGNN_B200_LIB=$PWD/paper_2402_08296_b200/variants/libpair.so python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"v":"edge_pair",/' >> $O
python tools/time_pcg.py 2>&1 | tail -1 >> $O
cat $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_c9.csv python tools/profile_pcg.py --iters 6 > gpurun_out/c9_launches.log 2>&1
tail -1 gpurun_out/c9_launches.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/c9_pytest.log 2>&1; tail -3 gpurun_out/c9_pytest.log
