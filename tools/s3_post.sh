# after the final pass: TC snapshot fix, Gram N trimmed to T, fp32 oz_w loading six R slots
O=gpurun_out/s3post
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
