#!/bin/bash
# round-2 cycle 3: GPU tests, H0-skip A/B, PCG timing, sharded bench (2 ranks on one
# GPU: gloo for setup, device-flag peer exchanges + CUDA graphs for the data path),
# per-iteration launch list, CPU PCG record at config B.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -x --durations=5 > gpurun_out/c3_pytest.log 2>&1
tail -8 gpurun_out/c3_pytest.log
O=gpurun_out/c3_ab.jsonl; : > $O
python tools/time_apply.py 2>&1 | tail -1 >> $O
DDMGNN_H0_SKIP=0 python tools/time_apply.py 2>&1 | tail -1 | sed 's/^{/{"h0_skip":0,/' >> $O
python tools/time_pcg.py 2>&1 | tail -1 >> $O
cat $O
for T in 100000 1000000; do
  DDMGNN_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 10 --warmup 3 \
    --target-nodes $T > gpurun_out/c3_sharded_$T.json 2> gpurun_out/c3_sharded_$T.err
  tail -c 1500 gpurun_out/c3_sharded_$T.json; tail -3 gpurun_out/c3_sharded_$T.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_pcg_launches_c3.csv python tools/profile_pcg.py --iters 6 > gpurun_out/r02_pcg_launches_c3.log 2>&1
timeout 900 python tools/cpu_pcg.py B gpurun_out/r02_cpu_pcg_B.json > gpurun_out/c3_cpu_pcg_B.log 2>&1
tail -c 600 gpurun_out/r02_cpu_pcg_B.json
