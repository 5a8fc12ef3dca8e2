import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', open(f).read()[-300:]); continue
    for k,v in d['per_config'].items():
        print(f.split('/')[-1], k, v['value'], v['ms_per_step'], 'chunks',v['chunks'], 'L',v['chunk_len'], 'frac', v['roofline']['frac'], {kk:round(x,3) for kk,x in v['kernels_ms'].items() if x>0.05})
