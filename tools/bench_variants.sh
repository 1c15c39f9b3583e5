#!/bin/bash
# Time every kernel variant build under paper_2402_08296_b200/variants/ against the main build.
mkdir -p gpurun_out
python tools/time_apply.py
for L in paper_2402_08296_b200/variants/*.so; do DDMGNN_B200_LIB=$PWD/$L python tools/time_apply.py; done
