cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "0 0 75776" "1 0 75776" "1 8 75776" "1 8 151552" "0 8 75776" "0 16 75776"; do
  set -- $v
  PAREM_CONV_TMA=$1 PAREM_CONV_REP=$2 PAREM_CONV_CHAINS=$3 timeout 300 python bench.py --config 3 --quick --steps 5 > gpurun_out/g23_tma$1_rep$2_ch$3.json 2>&1
done
PAREM_CONV_TMA=1 PAREM_CONV_REP=8 timeout 600 python -m pytest tests -m gpu -q -x -k "conv or config_small or configs_small" > gpurun_out/g23_tests.txt 2>&1
echo done
