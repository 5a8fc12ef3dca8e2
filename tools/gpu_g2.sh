cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ./tools/gather_probe > gpurun_out/g2_probe.txt 2>&1
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
echo done
