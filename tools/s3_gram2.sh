# ncu: single-CTA int8 Gram vs the CTA-pair kernel on cfg2-shaped data (8 subjects)
mkdir -p gpurun_out/s3g
python tools/gram_probe.py --config cfg2 --subjects 8 > gpurun_out/s3g/probe.log 2>&1
SRM_B200_GRAM_PAIRS=1 python tools/gram_probe.py --config cfg2 --subjects 8 >> gpurun_out/s3g/probe.log 2>&1
ncu --set full --clock-control none -k regex:"k_oz_gram" -s 0 -c 6 -f -o gpurun_out/s3g/gram1 python tools/gram_probe.py --config cfg2 --subjects 8 > gpurun_out/s3g/ncu1.log 2>&1
SRM_B200_GRAM_PAIRS=1 ncu --set full --clock-control none -k regex:"k_oz_gram" -s 0 -c 6 -f -o gpurun_out/s3g/gram2 python tools/gram_probe.py --config cfg2 --subjects 8 > gpurun_out/s3g/ncu2.log 2>&1
