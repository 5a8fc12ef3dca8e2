#!/bin/bash
# re-entry session: parity (gpu, not slow), default bench, launch list + ncu full of the top kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version,memory.total --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 > gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for k in 1 3 4 5; do timeout 600 python bench.py --config $k --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg$k.json 2> gpurun_out/bench_cfg$k.err; done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full $B > gpurun_out/ncu_full.log 2>&1
echo done
