#!/bin/bash
# A/B of the C1 frame rate between environment settings of one library
# (e.g. VF_PDL=0 VF_PDL=1), variants interleaved, three rounds.
for r in 1 2 3; do
for e in "$@"; do
  env $e python bench.py --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline --no-roofline-large ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$e', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['sync_value'],1), {k:round(v,4) for k,v in d['stage_ms'].items()})"
done; done
