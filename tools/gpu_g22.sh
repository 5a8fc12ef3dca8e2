cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g22_all.txt 2>&1
timeout 300 python bench.py --config 2 --steps 20 --no-enum --no-e2e --no-cpu-baseline --no-find > gpurun_out/g22_cfg2.json 2>&1
B="python bench.py --config 2 --quick --steps 2 --warmup 3"
$B > gpurun_out/g22_plain.json 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/g22_tiny $B > gpurun_out/g22_ncu.log 2>&1
echo done
