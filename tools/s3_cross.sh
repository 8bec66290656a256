# cross term from the polar + tail_kk beside apply_m (early_kk): parity, timelines, bench
mkdir -p gpurun_out/s3x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > gpurun_out/s3x/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/s3x/pytest_parity.log
for c in cfg2 cfg3; do
  timeout 600 python tools/chain_probe.py --config $c --out gpurun_out/s3x/chain_$c.json > gpurun_out/s3x/chain_$c.txt 2>&1
done
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3x/bench_cfg2.json 2> gpurun_out/s3x/bench_cfg2.err
timeout 1500 python -m pytest tests/test_gpu_baseline.py -x -q > gpurun_out/s3x/pytest_base.log 2>&1; echo "rc=$?" >> gpurun_out/s3x/pytest_base.log
