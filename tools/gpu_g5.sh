cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 3 5; do
  B="python bench.py --config $k --quick --steps 2 --warmup 3"
  $B > gpurun_out/g5_plain_$k.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_set|conv_follow" -s 8 -c 2 -o gpurun_out/g5_prof_cfg$k $B > gpurun_out/g5_ncu_$k.log 2>&1
done
echo done
