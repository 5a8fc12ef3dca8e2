cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PAREM_CONV_TMA=0 timeout 600 python -m pytest tests -m gpu -x -q -k "full_size and 4" > gpurun_out/g9_t4_notma.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -k "full_size" > gpurun_out/g9_full.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g9_all.txt 2>&1
echo done
