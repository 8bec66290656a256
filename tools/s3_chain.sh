# CUPTI kernel timelines of one bench step (cfg2/cfg3/cfg4) + ncu --set full of one eager cfg2 iteration
mkdir -p gpurun_out/s3c
for c in cfg2 cfg4 cfg3; do
  timeout 600 python tools/chain_probe.py --config $c --out gpurun_out/s3c/chain_$c.json > gpurun_out/s3c/chain_$c.txt 2>&1
done
timeout 900 ncu --profile-from-start off --set full --import-source on -f -o gpurun_out/s3c/iter_cfg2 \
  python tools/chain_probe.py --config cfg2 --eager > gpurun_out/s3c/ncu_iter.log 2>&1
