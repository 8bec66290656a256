# round-2 final measurement pass: every BASELINE config through bench.py (e2e + CPU sweep),
# the reference arm, the ncu launch list of the default command, one full capture of the
# dominant kernel (oz_gram, cfg2 shape), CUPTI timelines, then the GPU test suite and smoke()
set -x
O=gpurun_out/final6
mkdir -p $O
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/ref_cfg2.json 2> $O/ref_cfg2.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg2.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 600 python tools/gram_probe.py --config cfg2 --subjects 40 > $O/gp.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gram|k_oz_split" -s 2 -c 2 \
      -f -o $O/oz_cfg2 python tools/gram_probe.py --config cfg2 --subjects 40 > $O/ncu_oz.log 2>&1
for c in cfg2 cfg4; do
  timeout 600 python tools/chain_probe.py --config $c --out $O/chain_$c.json > $O/chain_$c.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
