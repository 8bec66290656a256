# 32x32 tail sweeps, fp32 final W via the tcgen05 A-pass, fp32 split 128 cols, NCCL exchange graph
mkdir -p gpurun_out/s3b
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fp32_final_w or nccl_exchange or eager_two_lane or batched_finalize or steps_match or errors" > gpurun_out/s3b/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/s3b/pytest_new.log
for c in cfg2 cfg4 cfg3 cfg5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3b/bench_$c.json 2> gpurun_out/s3b/bench_$c.err
done
SRM_B200_SPLIT_COLS=64 SRM_B200_FINAL_W=oz timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3b/bench_cfg4_old.json 2> gpurun_out/s3b/bench_cfg4_old.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_baseline.py -x -q > gpurun_out/s3b/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/s3b/pytest_all.log
