O=gpurun_out/s3wx
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "in_kernel_slicing or fp32 or int8_gram" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in cfg5 cfg4 cfg3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  SRM_B200_OZW=records timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_${c}_rec.json 2> $O/bench_${c}_rec.err
done
