# int8 Gram: off-diagonal tile pairs on CTA pairs + singles (SRM_B200_GRAM_PAIRS=1) vs single CTAs
mkdir -p gpurun_out/s3p
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cta_pairs" > gpurun_out/s3p/pytest_pairs.log 2>&1; echo "rc=$?" >> gpurun_out/s3p/pytest_pairs.log
for c in cfg2 cfg4 cfg3; do
  SRM_B200_GRAM_PAIRS=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3p/bench_${c}_pairs.json 2> gpurun_out/s3p/bench_${c}_pairs.err
  SRM_B200_GRAM_PAIRS=0 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3p/bench_${c}_single.json 2> gpurun_out/s3p/bench_${c}_single.err
done
