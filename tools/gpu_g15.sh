cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_batch_gpu.py -q -x > gpurun_out/g15_batch.txt 2>&1
timeout 300 python bench.py --config 1 --steps 20 > gpurun_out/g15_cfg1.json 2> gpurun_out/g15_cfg1.err
echo done
