#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_merge $B > gpurun_out/ncu_full2.log 2>&1
B3="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lanes_kernel -s 3 -c 1 -o gpurun_out/prof_cfg3 $B3 > gpurun_out/ncu_full3.log 2>&1
python tools/quick_time.py 4 5 > gpurun_out/qt45.log 2>&1
echo done
