cd $GRAFT_REPO_ROOT; out=gpurun_out/hy3; mkdir -p $out
run() { # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --config 5 --quick --steps 5 --warmup 3 --verify > $out/$name.json 2> $out/$name.err
}
run hyb_cpt2_512 PAREM_CONV_HYB=1
run hyb_cpt1_512 PAREM_CONV_HYB=1 PAREM_CONV_CPT=1
run hyb_cpt2_384 PAREM_CONV_HYB=1 PAREM_CONV_FTHREADS=384
run hyb_cpt2_320 PAREM_CONV_HYB=1 PAREM_CONV_FTHREADS=320
run plain_cpt2_256 PAREM_CONV_CPT=2 PAREM_CONV_FTHREADS=256 PAREM_CONV_CHAINS=75776
run plain_cpt2_512 PAREM_CONV_CPT=2 PAREM_CONV_FTHREADS=512 PAREM_CONV_CHAINS=151552
PAREM_CONV_HYB=1 timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "conv" > $out/pytest_hyb.txt 2>&1
echo done > $out/status.txt
