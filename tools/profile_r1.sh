#!/bin/bash
# Profiling recipe (runs on the GPU box under gpurun). Outputs into gpurun_out/.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"k_icp|k_raycast|k_integrate_s|k_mark|k_alloc_compact|k_alloc_apply|k_visible|k_ranges|k_pyramid" \
    -s 40 -c 10 -o gpurun_out/prof_c1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err
python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
ncu --set full --import-source on --clock-control none -k regex:"k_integrate_s" -s 6 -c 1 \
    -o gpurun_out/prof_c3_integrate python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
