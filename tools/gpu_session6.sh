#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for k in 1 3 5 4; do timeout 600 python bench.py --config $k --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg$k.json 2> gpurun_out/bench_cfg$k.err; done
echo done
