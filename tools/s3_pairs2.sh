# fp32: CTA-pair Gram tiles beside the single tiles in each batch (default) vs single CTAs
mkdir -p gpurun_out/s3q
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cta_pairs or int8_gram_fp32 or fp32_configs" > gpurun_out/s3q/pytest_pairs.log 2>&1; echo "rc=$?" >> gpurun_out/s3q/pytest_pairs.log
for c in cfg4 cfg3 cfg5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3q/bench_${c}_pairs.json 2> gpurun_out/s3q/bench_${c}_pairs.err
  SRM_B200_GRAM_PAIRS=0 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3q/bench_${c}_single.json 2> gpurun_out/s3q/bench_${c}_single.err
done
