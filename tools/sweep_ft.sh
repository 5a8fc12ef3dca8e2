cd $GRAFT_REPO_ROOT; out=gpurun_out/ft2; mkdir -p $out
run() { name=$1; k=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $k --quick --steps 5 --warmup 3 > $out/$name.json 2> $out/$name.err
}
run cfg4_base 4 X=1
run cfg4_d2 4 PAREM_CONV_DMAX=2
run cfg4_ft288 4 PAREM_CONV_FTHREADS=288 PAREM_CONV_CHAINS=42624
run cfg4_ft352 4 PAREM_CONV_FTHREADS=352 PAREM_CONV_CHAINS=52096
run cfg4_ft320_d2 4 PAREM_CONV_FTHREADS=320 PAREM_CONV_CHAINS=47360 PAREM_CONV_DMAX=2
run cfg5_d2 5 PAREM_CONV_DMAX=2
run cfg3_d2 3 PAREM_CONV_DMAX=2
echo done > $out/status.txt
