#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 3 5 4; do
  for la in 0 16 64; do
    PAREM_CONV_LADD=$la timeout 300 python bench.py --config $k --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$k', 'ladd=$la L=', d['config']['chunk_len'], d['value'], {k: round(v,3) for k,v in d['kernels_ms'].items()})"
  done
done
for k in 3 5; do
  PAREM_CONV_CHAINS=37888 timeout 300 python bench.py --config $k --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$k', 'chains 37888 L=', d['config']['chunk_len'], d['value'], {k: round(v,3) for k,v in d['kernels_ms'].items()})"
done
