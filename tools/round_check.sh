#!/bin/bash
# Full round check on the GPU box (under gpurun): GPU tests, smoke, bench lines, launch list, ncu captures.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c1.json 2> gpurun_out/bench_ref_c1.err
timeout 600 python bench.py --config C2 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
timeout 600 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err
timeout 900 python bench.py --config C4 --steps 995 --warmup 5 > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err
timeout 600 python bench.py --config C2L --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2l.json 2>gpurun_out/bench_c2l.err
timeout 600 python bench.py --config C1R > gpurun_out/bench_c1r.json 2>gpurun_out/bench_c1r.err
timeout 600 python bench.py --config C2T > gpurun_out/bench_c2t.json 2>gpurun_out/bench_c2t.err
if [ -z "$SKIP_NCU" ]; then
timeout 900 bash tools/profile_r1.sh > gpurun_out/profile.log 2>&1
fi
