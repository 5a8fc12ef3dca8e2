cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/find_once.py 2 > gpurun_out/g18_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"find_emit|tiny_kernel" -s 2 -c 2 -o gpurun_out/g18_emit python tools/find_once.py 2 > gpurun_out/g18_ncu.log 2>&1
echo done
