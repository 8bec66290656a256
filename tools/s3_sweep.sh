# sweep without per-element selects (per-R kernels), tail_s on 16 warps, ns_polar_g cp.async
mkdir -p gpurun_out/s3w
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > gpurun_out/s3w/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3w/pytest.log
for c in cfg2 cfg3; do
  timeout 600 python tools/chain_probe.py --config $c --out gpurun_out/s3w/chain_$c.json > gpurun_out/s3w/chain_$c.txt 2>&1
done
timeout 900 ncu --profile-from-start off --set full --import-source on -f -o gpurun_out/s3w/iter_cfg3 \
  python tools/chain_probe.py --config cfg3 --eager > gpurun_out/s3w/ncu_iter.log 2>&1
