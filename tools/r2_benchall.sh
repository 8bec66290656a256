set -x
mkdir -p gpurun_out/r2
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err; done
python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2/ref_cfg2.json 2> gpurun_out/r2/ref_cfg2.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_launch.log 2>&1
