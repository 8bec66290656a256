# session 7: the remaining BASELINE configs and the reference arm at HEAD (completes profiles/r2s7)
set -x
O=gpurun_out/final7
mkdir -p $O
for c in cfg1 cfg4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/ref_cfg2.json 2> $O/ref_cfg2.err
for c in cfg2 cfg4; do
  timeout 600 python tools/chain_probe.py --config $c --out $O/chain_$c.json > $O/chain_$c.txt 2>&1
done
ls -la $O
