cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ./tools/gather_probe > gpurun_out/g6_probe.txt 2>&1
for k in 3; do
  timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g6_cfg$k.json 2>&1
  PAREM_CONV_CPT=2 timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g6_cfg${k}_cpt2.json 2>&1
  PAREM_CONV_CPT=2 PAREM_CONV_CHAINS=303104 timeout 300 python bench.py --config $k --quick --steps 5 > gpurun_out/g6_cfg${k}_cpt2_ch303.json 2>&1
done
PAREM_CONV_CHAINS=75776 PAREM_CONV_CPT=1 timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g6_cfg5_ch75.json 2>&1
echo done
