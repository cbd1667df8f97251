#!/bin/bash
# A/B: default bench (C1 line + the C3/C2L integration roofline leg) with each library variant
for v in "$@"; do
  VOXFUSE_B200_LIB=$v/libvoxfuse_b200.so python bench.py --steps 30 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} | python -c "
import json,sys; d=json.loads(sys.stdin.read()); L=d['roofline'].get('large',{})
print('$v', round(d['value'],1), {k:round(v,4) for k,v in d['stage_ms'].items()}, {k:(round(L[k]['ms_per_launch'],4), round(L[k]['frac'],3)) for k in ('exact','fast','exact_rgb','fast_rgb') if k in L})"
done
