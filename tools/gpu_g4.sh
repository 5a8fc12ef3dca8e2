cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g4_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/g4_tests.txt
for k in 3 5 4; do
  timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g4_cfg$k.json 2> gpurun_out/g4_cfg$k.err
done
for ch in 151552 303104 606208; do
  PAREM_CONV_CHAINS=$ch timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g4_cfg5_ch$ch.json 2>&1
done
PAREM_CONV_CPT=1 timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g4_cfg5_cpt1.json 2>&1
for hx in 4 8; do PAREM_CONV_HEADX=$hx timeout 300 python bench.py --config 4 --quick --steps 5 > gpurun_out/g4_cfg4_hx$hx.json 2>&1; done
for ch in 75776 303104; do PAREM_CONV_CHAINS=$ch timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g4_cfg3_ch$ch.json 2>&1; done
PAREM_CONV_REP=0 timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g4_cfg3_rep0.json 2>&1
echo done
