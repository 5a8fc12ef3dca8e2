cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=$(date +%s)
timeout 900 python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
echo "bench $(( $(date +%s) - S )) s" > gpurun_out/g3_times.txt
for k in 3 5 4; do
  B="python bench.py --config $k --quick --steps 3 --warmup 3"
  $B > gpurun_out/g3_plain_$k.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_set|conv_follow" -s 6 -c 2 -o gpurun_out/g3_prof_cfg$k $B > gpurun_out/g3_ncu_$k.log 2>&1
  echo "cfg$k $(( $(date +%s) - S )) s" >> gpurun_out/g3_times.txt
done
echo done
