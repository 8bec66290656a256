mkdir -p gpurun_out/s3q2
for rep in 1 2; do
SRM_B200_GRAM_PAIRS=1 timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3q2/bench_cfg2_pairs_$rep.json 2> gpurun_out/s3q2/bench_cfg2_pairs_$rep.err
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3q2/bench_cfg2_single_$rep.json 2> gpurun_out/s3q2/bench_cfg2_single_$rep.err
done
