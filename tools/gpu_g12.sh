cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 5 4; do
  timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g12_cfg$k.json 2>&1
done
echo done
