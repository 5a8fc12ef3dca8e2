# final evidence for this round: default bench line, launch lists, ncu --set full of every
# config's dominant kernels (each ncu run after the same command exited 0 without ncu),
# GPU tests and the randomised stress.  The ncu reports are summarised on the box
# (tools/ncu_json.py) and deleted: gpurun copies back at most 64 MiB.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final; F=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $F/gpu.txt
timeout 1200 python bench.py > $F/bench.json 2> $F/bench.err
echo "bench rc=$?" > $F/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $F/pytest.txt 2>&1
echo "pytest rc=$?" >> $F/status.txt
for k in 5 4 3; do
  B="python bench.py --config $k --quick --steps 3 --warmup 3"
  $B > $F/plain_$k.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_cfg$k.csv $B > $F/ncu_launch_$k.log 2>&1
done
for k in 3 4 5; do
  B="python bench.py --config $k --quick --steps 1 --warmup 3"
  $B > $F/plain1_$k.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_set|conv_follow" -s 6 -c 2 -o $F/prof_cfg$k $B > $F/ncu_full_$k.log 2>&1
  for kn in conv_set conv_follow; do
    python tools/ncu_json.py $F/prof_cfg$k.ncu-rep "${kn}" $F/r02_ncu_full_cfg${k}_${kn}.json "tools/gpu_final.sh: ncu --set full --clock-control none, bench.py --config $k --quick --steps 1 (round-2 final code)" > /dev/null 2>&1
  done
  rm -f $F/prof_cfg$k.ncu-rep
done
for k in 2 1; do
  B="python bench.py --config $k --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-find --no-enum --no-lanes"
  $B > $F/plain_t$k.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o $F/prof_cfg$k $B > $F/ncu_full_$k.log 2>&1
  python tools/ncu_json.py $F/prof_cfg$k.ncu-rep "tiny_kernel" $F/r02_ncu_full_cfg${k}_tiny.json "tools/gpu_final.sh: ncu --set full --clock-control none, bench.py --config $k (round-2 final code)" > /dev/null 2>&1
  rm -f $F/prof_cfg$k.ncu-rep
done
STRESS_BASE=900000 timeout 1500 python tools/stress.py 1000 > $F/stress.txt 2>&1
echo done >> $F/status.txt
