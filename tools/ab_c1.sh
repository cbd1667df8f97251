#!/bin/bash
# A/B of the C1 frame rate only (no roofline leg), long runs, variants interleaved
for r in 1 2 3; do
for v in "$@"; do
  VOXFUSE_B200_LIB=$v/libvoxfuse_b200.so python bench.py --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline --no-roofline-large ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', round(d['value'],1), round(d['e2e']['value'],1), {k:round(v,4) for k,v in d['stage_ms'].items()})"
done; done
