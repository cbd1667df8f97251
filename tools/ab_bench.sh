#!/bin/bash
# A/B: bench C1 with each library variant given as argument (dirs containing libvoxfuse_b200.so)
for v in "$@"; do
  VOXFUSE_B200_LIB=$v/libvoxfuse_b200.so python bench.py --steps 30 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k:round(v,4) for k,v in d['stage_ms'].items()})"
done
