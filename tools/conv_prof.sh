#!/bin/bash
# ncu --set full of the converging path's kernels (cfg3 by default)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K=${1:-3}
B="python bench.py --config $K --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain_cfg$K.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_ -s 8 -c 4 -o gpurun_out/prof_conv_cfg$K $B > gpurun_out/ncu_conv_cfg$K.log 2>&1
echo done
