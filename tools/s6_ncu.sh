# session 6: ncu launch list of the default command (our kernels: -k regex:k_) and full captures of the
# dominant kernel and of the kernels changed this session (group-walking slicing, final W with tiled
# R'^T slices, slot-pair init term) on cfg 2, and the final W on a cfg 5 slice
set -x
O=gpurun_out/final6
mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/launches_cfg2.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gram" -s 1 -c 1 \
      -f -o $O/oz_gram_cfg2 python tools/gram_probe.py --config cfg2 --subjects 40 > $O/ncu_oz.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_split" -s 12 -c 1 \
      -f -o $O/oz_split_cfg2 python tools/gram_probe.py --config cfg2 --subjects 40 > $O/ncu_split.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_rowgemm|k_oz_nt" -c 2 \
    -f -o $O/ozw_nt_cfg2 python bench.py --config cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_ozw2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_rowgemm" -c 1 \
    -f -o $O/ozw_cfg5 python bench.py --config cfg5 --subjects 16 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_ozw5.log 2>&1
ls -la $O/*.ncu-rep
