#!/bin/bash
# per-kernel launch times of the converging path (cfg3, cfg5, cfg4) + the tiny kernel (cfg2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 3 5 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$k.csv \
    python bench.py --config $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/ncu_launch_cfg$k.log 2>&1
done
