cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PAREM_CONV_TMA=1 PAREM_CONV_REP=8
B="python bench.py --config 3 --quick --steps 2 --warmup 3"
$B > gpurun_out/g24_plain.json 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_follow -s 3 -c 1 -o gpurun_out/g24_rep8 $B > gpurun_out/g24_ncu.log 2>&1
echo done
