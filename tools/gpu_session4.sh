#!/bin/bash
# full-size parity (BASELINE configs) + bench + ncu evidence for the default bench command
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version,memory.total --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 > gpurun_out/lscpu.txt
timeout 1200 python -m pytest tests -q -m "slow" -x > gpurun_out/pytest_slow.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slow.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full $B > gpurun_out/ncu_full.log 2>&1
echo done
