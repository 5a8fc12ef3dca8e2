cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g14_all.txt 2>&1
timeout 900 python bench.py > gpurun_out/g14_bench.json 2> gpurun_out/g14_bench.err
echo done
