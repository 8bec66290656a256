# ns_polar_g with cp.async staging: parity of the kp > 80 paths, cfg3 timeline
mkdir -p gpurun_out/s3n
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -k "wide_k or fp32_configs or exact or polar or cfg3 or int8_gram_fp32" > gpurun_out/s3n/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3n/pytest.log
timeout 600 python tools/chain_probe.py --config cfg3 --out gpurun_out/s3n/chain_cfg3.json > gpurun_out/s3n/chain_cfg3.txt 2>&1
timeout 600 python tools/chain_probe.py --config cfg5 --out gpurun_out/s3n/chain_cfg5.json > gpurun_out/s3n/chain_cfg5.txt 2>&1
