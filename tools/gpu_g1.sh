cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/g1_gpu.txt
nproc > gpurun_out/g1_nproc.txt; lscpu > gpurun_out/g1_lscpu.txt 2>&1
timeout 300 ./tools/gather_probe > gpurun_out/g1_probe.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.txt 2>&1
echo done
