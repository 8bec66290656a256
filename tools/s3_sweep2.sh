mkdir -p gpurun_out/s3v
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > gpurun_out/s3v/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3v/pytest.log
for c in cfg2 cfg3; do
  timeout 600 python tools/chain_probe.py --config $c --out gpurun_out/s3v/chain_$c.json > gpurun_out/s3v/chain_$c.txt 2>&1
done
for c in cfg2 cfg5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3v/bench_$c.json 2> gpurun_out/s3v/bench_$c.err
done
