#!/bin/bash
# final round-1 evidence: default bench line, launch list + ncu full of the headline kernel,
# conv_follow (cfg3, cfg5) and conv_set (cfg4) captures, bench lines of every config
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version,memory.total --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for k in 1 3 5 4; do timeout 600 python bench.py --config $k --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_cfg$k.json 2> gpurun_out/bench_cfg$k.err; done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --no-find --no-graph"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full $B > gpurun_out/ncu_full.log 2>&1
for k in 3 5; do
  B3="python bench.py --config $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --no-find"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_follow -s 3 -c 1 -o gpurun_out/prof_cfg${k}_follow $B3 > gpurun_out/ncu_follow$k.log 2>&1
done
B4="python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --no-find"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_set -s 3 -c 1 -o gpurun_out/prof_cfg4_set $B4 > gpurun_out/ncu_set4.log 2>&1
echo done
