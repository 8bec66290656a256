# tail_var (eigenbasis E-step tail) validation: parity suites + cfg2/cfg3 bench
mkdir -p gpurun_out/s3t
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -k "eigenbasis" > gpurun_out/s3t/pytest_eig.log 2>&1; timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > gpurun_out/s3t/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/s3t/pytest_parity.log
timeout 900 python -m pytest tests/test_gpu_baseline.py -x -q -k "cfg1 or cfg2 or cfg3" > gpurun_out/s3t/pytest_base.log 2>&1; echo "rc=$?" >> gpurun_out/s3t/pytest_base.log
for c in cfg2 cfg3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3t/bench_$c.json 2> gpurun_out/s3t/bench_$c.err
done
