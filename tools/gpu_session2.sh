#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_tma $B > gpurun_out/ncu_full.log 2>&1
echo done
