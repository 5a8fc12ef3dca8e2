# final evidence for this round: default bench line, launch lists, ncu --set full of every
# config's dominant kernels (each ncu run after the same command exited 0 without ncu),
# GPU tests and the randomised stress
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/final/gpu.txt
timeout 1200 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
echo "bench rc=$?" > gpurun_out/final/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/final/status.txt
for k in 5 4 3; do
  B="python bench.py --config $k --quick --steps 3 --warmup 3"
  $B > gpurun_out/final/plain_$k.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_cfg$k.csv $B > gpurun_out/final/ncu_launch_$k.log 2>&1
done
for k in 3 4 5; do
  B="python bench.py --config $k --quick --steps 1 --warmup 3"
  $B > gpurun_out/final/plain1_$k.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_set|conv_follow" -s 6 -c 2 -o gpurun_out/final/prof_cfg$k $B > gpurun_out/final/ncu_full_$k.log 2>&1
done
STRESS_BASE=700000 timeout 1500 python tools/stress.py 1000 > gpurun_out/final/stress.txt 2>&1
echo done >> gpurun_out/final/status.txt
