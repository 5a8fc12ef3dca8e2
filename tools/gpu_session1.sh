#!/bin/bash
# first measurement session: parity, bench, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2 $B > gpurun_out/ncu_full.log 2>&1
echo done
