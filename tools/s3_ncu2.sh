# launch list of the default bench command (our kernels only) + one full capture of oz_gram / oz_split (cfg2 shape)
O=gpurun_out/s3ncu
mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/launches_cfg2.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gram" -s 1 -c 1 \
      -f -o $O/oz_gram_cfg2 python tools/gram_probe.py --config cfg2 --subjects 40 > $O/ncu_oz.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_split" -s 12 -c 1 \
      -f -o $O/oz_split_cfg2 python tools/gram_probe.py --config cfg2 --subjects 40 > $O/ncu_split.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py tests/test_gpu_kernels.py tests/test_multirank.py -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
