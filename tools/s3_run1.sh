mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3/pytest_gpu.log
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench_$c.json 2> gpurun_out/s3/bench_$c.err
done
