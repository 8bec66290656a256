# rotated iteration graph + C = var_s + column-block exchange: tests, timelines, bench, ncu of the cfg3 iteration
mkdir -p gpurun_out/s3r
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_multirank.py -x -q > gpurun_out/s3r/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3r/pytest.log
for c in cfg2 cfg3; do
  timeout 600 python tools/chain_probe.py --config $c --out gpurun_out/s3r/chain_$c.json > gpurun_out/s3r/chain_$c.txt 2>&1
done
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3r/bench_cfg2.json 2> gpurun_out/s3r/bench_cfg2.err
timeout 900 ncu --profile-from-start off --set full --import-source on -f -o gpurun_out/s3r/iter_cfg3 \
  python tools/chain_probe.py --config cfg3 --eager > gpurun_out/s3r/ncu_iter.log 2>&1
