#!/bin/bash
# sanitizers on the round-2 code paths + 4 / 8 ranks sharing the GPU (functional check
# of the device-flag exchanges with the driver's scaling rank counts)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "apply or pcg" > gpurun_out/c15_memcheck.log 2>&1
tail -4 gpurun_out/c15_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "config_a" > gpurun_out/c15_racecheck.log 2>&1
tail -4 gpurun_out/c15_racecheck.log
for N in 4 8; do
  DDMGNN_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 5 --warmup 3 \
    --target-nodes 100000 > gpurun_out/c15_sharded_$N.json 2> gpurun_out/c15_sharded_$N.err
  tail -c 700 gpurun_out/c15_sharded_$N.json; grep -i "error\|Traceback" gpurun_out/c15_sharded_$N.err | head -3
done
