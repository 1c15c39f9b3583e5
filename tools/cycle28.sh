#!/bin/bash
# Records with the dataflow kernel: config D (10M DOFs, 1 GPU) and the config E sweep.
mkdir -p gpurun_out
timeout 1500 python bench.py --target-nodes 10000000 --no-cpu --steps 10 --warmup 3 > gpurun_out/c28_configD.json 2> gpurun_out/c28_configD.err
tail -c 400 gpurun_out/c28_configD.json; tail -3 gpurun_out/c28_configD.err
timeout 1800 python tools/sweep.py --min-nodes 1000000 > gpurun_out/c28_sweep.jsonl 2> gpurun_out/c28_sweep.err
wc -l gpurun_out/c28_sweep.jsonl; tail -2 gpurun_out/c28_sweep.err
