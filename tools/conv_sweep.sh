#!/bin/bash
# converging path: chunk-length sweep (K1 set walk vs K2 follow balance)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 3 5 4; do
  for L in 0 28352 56704 113408; do
    timeout 300 python bench.py --config $k --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --chunk-len $L 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$k', 'L=', d['config']['chunk_len'], 'p=', d['config']['chunks'], d['value'], {k: round(v,3) for k,v in d['kernels_ms'].items()})"
  done
done
