cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g10_all.txt 2>&1
for k in 3 5 4; do
  timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g10_cfg$k.json 2>&1
done
PAREM_CONV_CHAINS=75776 timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g10_cfg5_ch75.json 2>&1
PAREM_CONV_CHAINS=227328 timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g10_cfg3_ch227.json 2>&1
echo done
