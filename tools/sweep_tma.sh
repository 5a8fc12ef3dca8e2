cd $GRAFT_REPO_ROOT; out=gpurun_out/tm1; mkdir -p $out
run() { name=$1; k=$2; shift; shift
  env "$@" timeout 300 python bench.py --config $k --quick --steps 5 --warmup 3 --verify > $out/$name.json 2> $out/$name.err
}
run cfg3_tma_512 3 PAREM_CONV_TMA=1 PAREM_CONV_CHAINS=75776
run cfg3_tma_1024 3 PAREM_CONV_TMA=1
run cfg3_tma_rep8_512 3 PAREM_CONV_TMA=1 PAREM_CONV_REP=8 PAREM_CONV_CHAINS=75776
run cfg3_tma_rep8_1024 3 PAREM_CONV_TMA=1 PAREM_CONV_REP=8
run cfg3_tma_768 3 PAREM_CONV_TMA=1 PAREM_CONV_CHAINS=113664
echo done > $out/status.txt
