# final evidence for this round: default bench line, launch lists, ncu --set full of every
# config's dominant kernels (each ncu run after the same command exited 0 without ncu)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/final/gpu.txt
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
echo "bench rc=$?" > gpurun_out/final/status.txt
for k in 5 3; do
  B="python bench.py --config $k --quick --steps 3 --warmup 3"
  $B > gpurun_out/final/plain_$k.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_cfg$k.csv $B > gpurun_out/final/ncu_launch_$k.log 2>&1
done
for k in 3 4 5; do
  B="python bench.py --config $k --quick --steps 1 --warmup 3"
  $B > gpurun_out/final/plain1_$k.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_set|conv_follow" -s 6 -c 2 -o gpurun_out/final/prof_cfg$k $B > gpurun_out/final/ncu_full_$k.log 2>&1
done
B="python bench.py --config 1 --quick --steps 2 --warmup 3"
$B > gpurun_out/final/plain_1.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/final/prof_cfg1 $B > gpurun_out/final/ncu_full_1.log 2>&1
echo done >> gpurun_out/final/status.txt
