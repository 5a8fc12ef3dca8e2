cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "find or position or host" > gpurun_out/g17_find.txt 2>&1
timeout 300 python bench.py --config 2 --steps 20 > gpurun_out/g17_cfg2.json 2> gpurun_out/g17_cfg2.err
timeout 300 python bench.py --config 4 --steps 5 --no-enum --no-find --no-cpu-baseline > gpurun_out/g17_cfg4.json 2> gpurun_out/g17_cfg4.err
echo done
