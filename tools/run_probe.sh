cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/pb1
timeout 300 ./build/follow_probe > gpurun_out/pb1/follow_probe5.txt 2>&1
for k in 4 5 3; do
  timeout 300 python bench.py --config $k --quick --steps 5 --warmup 3 > gpurun_out/pb1/cfg${k}.json 2> gpurun_out/pb1/cfg${k}.err
done
echo done > gpurun_out/pb1/status.txt
