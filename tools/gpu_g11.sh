cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 3 5 4; do
  timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g11_cfg$k.json 2>&1
  PAREM_SET_OWN=0 timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g11_cfg${k}_bm.json 2>&1
done
PAREM_CONV_CHAINS=151552 timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g11_cfg5_ch151.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "conv or config" > gpurun_out/g11_tests.txt 2>&1
echo done
