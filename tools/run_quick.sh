# quick GPU session: bench (5 steps) + GPU tests; outputs under gpurun_out/$1
cd $GRAFT_REPO_ROOT; out=gpurun_out/${1:-q}; mkdir -p $out
for k in ${CFGS:-4 5 3}; do
  timeout 300 python bench.py --config $k --quick --steps 5 --warmup 3 > $out/cfg${k}.json 2> $out/cfg${k}.err
done
PAREM_CONV_CPT=2 PAREM_CONV_FTHREADS=512 PAREM_CONV_CHAINS=151552 timeout 300 python bench.py --config 3 --quick --steps 5 --warmup 3 > $out/cfg3_cpt2_512.json 2> $out/cfg3_cpt2_512.err
PAREM_CONV_CPT=2 PAREM_CONV_FTHREADS=256 PAREM_CONV_CHAINS=75776 timeout 300 python bench.py --config 3 --quick --steps 5 --warmup 3 > $out/cfg3_cpt2_256.json 2> $out/cfg3_cpt2_256.err
PAREM_CONV_CPT=2 PAREM_CONV_FTHREADS=384 PAREM_CONV_CHAINS=113664 timeout 300 python bench.py --config 3 --quick --steps 5 --warmup 3 > $out/cfg3_cpt2_384.json 2> $out/cfg3_cpt2_384.err
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $out/pytest.txt 2>&1; fi
echo done > $out/status.txt
