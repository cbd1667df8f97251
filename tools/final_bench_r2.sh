set -x
python bench.py > gpurun_out/r2f_bench_c1.json 2> gpurun_out/r2f_bench_c1.err
for cfg in C3 C2 C2L C4 C4B100 C4R C1R C2T; do
  python bench.py --config $cfg --no-cpu-baseline --no-roofline-large > gpurun_out/r2f_bench_$cfg.json 2> gpurun_out/r2f_bench_$cfg.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches_c1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-roofline-large > gpurun_out/r2f_ncu.log 2>&1
