#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in 7104 7168 7232 7296 7360; do
  timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --chunk-len $L 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 L=', d['config']['chunk_len'], 'p=', d['config']['chunks'], 'grid', d['config']['grid'], d['value'], d['kernels_ms'])"
done
for L in 56688 56704 56720 56736 56752 56784 56816 56848; do
  timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --chunk-len $L 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 L=', d['config']['chunk_len'], d['value'], round(d['kernels_ms']['conv_follow'],3))"
done
