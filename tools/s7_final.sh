# session 7 final pass at HEAD (final W: both feature halves of an item on one CTA): default bench line,
# the kp = 128 configs the change touches, the reference arm, then the whole GPU suite and smoke()
set -x
O=gpurun_out/final7
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
tail -3 $O/pytest_gpu.log $O/smoke.log
