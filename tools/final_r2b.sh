# round-2 final: GPU suite, smoke, bench lines of every config, launch list of the default bench
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final2.txt 2>&1; tail -2 gpurun_out/gputests_final2.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.txt 2>&1; echo smoke rc $?
python bench.py > gpurun_out/r2h_bench_c1.json 2>/dev/null
for cfg in C3 C2 C2L C4 C4B100 C4R C1R C2T; do
  python bench.py --config $cfg --no-cpu-baseline --no-roofline-large > gpurun_out/r2h_bench_$cfg.json 2>/dev/null
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches_c1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-roofline-large > /dev/null 2>&1
echo done
