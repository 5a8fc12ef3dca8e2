#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 3 5 4; do
  for ch in 151552 75776; do
    for dm in 1 2 4; do
      PAREM_CONV_CHAINS=$ch PAREM_CONV_DMAX=$dm timeout 300 python bench.py --config $k --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$k', 'chains=$ch dmax=$dm L=', d['config']['chunk_len'], d['value'], {k: round(v,3) for k,v in d['kernels_ms'].items()})"
    done
  done
done
