cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "conv or config" > gpurun_out/g8_tests.txt 2>&1
for k in 3 5 4; do
  timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g8_cfg$k.json 2>&1
done
PAREM_CONV_CHAINS=75776 timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g8_cfg3_ch75.json 2>&1
PAREM_CONV_CHAINS=75776 timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g8_cfg5_ch75.json 2>&1
PAREM_CONV_CHAINS=303104 timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g8_cfg5_ch303.json 2>&1
PAREM_CONV_TMA=0 timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g8_cfg3_notma.json 2>&1
echo done
