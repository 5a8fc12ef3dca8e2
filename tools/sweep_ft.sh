cd $GRAFT_REPO_ROOT; out=gpurun_out/ft1; mkdir -p $out
for k in 4 5; do
  for ft in 256 320 384 448; do
    ch=$((148*ft))
    PAREM_CONV_FTHREADS=$ft PAREM_CONV_CHAINS=$ch timeout 300 python bench.py --config $k --quick --steps 5 --warmup 3 > $out/cfg${k}_ft${ft}.json 2> $out/cfg${k}_ft${ft}.err
  done
done
echo done > $out/status.txt
