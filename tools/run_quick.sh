# quick GPU session: bench (5 steps) + GPU tests; outputs under gpurun_out/$1
cd $GRAFT_REPO_ROOT; out=gpurun_out/${1:-q}; mkdir -p $out
for k in ${CFGS:-4 5 3}; do
  timeout 300 python bench.py --config $k --quick --steps 5 --warmup 3 --verify > $out/cfg${k}.json 2> $out/cfg${k}.err
done
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $out/pytest.txt 2>&1; fi
echo done > $out/status.txt
