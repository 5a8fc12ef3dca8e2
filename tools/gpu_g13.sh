cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for ch in 113664 151552 189440; do PAREM_CONV_CHAINS=$ch timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g13_cfg3_tma_$ch.json 2>&1; done
for ch in 75776 113664; do PAREM_CONV_TMA=0 PAREM_CONV_CHAINS=$ch timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g13_cfg3_notma_$ch.json 2>&1; done
timeout 300 python bench.py --config 5 --quick --steps 5 > gpurun_out/g13_cfg5.json 2>&1
echo done
