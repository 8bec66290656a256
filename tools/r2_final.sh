# round-2 measurement pass: every BASELINE config through bench.py (e2e + CPU sweep),
# the reference arm, the ncu launch list of the default command and one full
# capture of the dominant kernel, then the GPU test suite and smoke()
set -x
mkdir -p gpurun_out/final
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/final/ref_cfg2.json 2> gpurun_out/final/ref_cfg2.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final/launches_cfg2.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_launch.log 2>&1
python tools/gram_probe.py --config cfg2 --subjects 40 > gpurun_out/final/gp.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_oz_gram|k_oz_nt|k_oz_split" -s 3 -c 3 \
      -o gpurun_out/final/oz_cfg2 python tools/gram_probe.py --config cfg2 --subjects 40 > gpurun_out/final/ncu_oz.log 2>&1
