mkdir -p gpurun_out/s3c
timeout 900 ncu --profile-from-start off --set full --import-source on -f -o gpurun_out/s3c/iter_cfg2 \
  python tools/chain_probe.py --config cfg2 --eager > gpurun_out/s3c/ncu_iter.log 2>&1
tail -3 gpurun_out/s3c/ncu_iter.log
