#!/bin/bash
# round-2 cycle 2: GPU tests (device-flag sharded path, fused PCG tail, ALU relu),
# A/B timings, launch list of the PCG iteration.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -x --durations=8 > gpurun_out/c2_pytest.log 2>&1
tail -15 gpurun_out/c2_pytest.log
O=gpurun_out/c2_ab.jsonl; : > $O
python tools/time_apply.py >> $O 2>&1
DDMGNN_B200_LIB=$PWD/paper_2402_08296_b200/variants/librelu0.so python tools/time_apply.py 2>&1 | tail -1 >> $O
python tools/time_pcg.py 2>&1 | tail -1 >> $O
DDMGNN_FUSED_TAIL=0 python tools/time_pcg.py 2>&1 | tail -1 >> $O
cat $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_fused.csv python tools/profile_pcg.py --iters 6 > gpurun_out/r02_pcg_launches_fused.log 2>&1
tail -2 gpurun_out/r02_pcg_launches_fused.log
