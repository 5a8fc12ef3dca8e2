#!/bin/bash
# round-1 ncu evidence: cfg2 launch list + full capture of the tiny kernel; cfg3/cfg5 full
# captures of the converging path's set-walk and follow kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full $B > gpurun_out/ncu_full.log 2>&1
for k in 3 5; do
  B3="python bench.py --config $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_follow -s 3 -c 1 -o gpurun_out/prof_cfg${k}_follow $B3 > gpurun_out/ncu_follow$k.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_set -s 3 -c 1 -o gpurun_out/prof_cfg${k}_set $B3 > gpurun_out/ncu_set$k.log 2>&1
done
echo done
