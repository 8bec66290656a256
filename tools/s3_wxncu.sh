O=gpurun_out/s3wxn
mkdir -p $O
timeout 600 python tools/gram_probe.py --config cfg4 --subjects 16 --finalize > $O/probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_rowgemm" -s 2 -c 1 -f -o $O/wx_cfg4 \
   python tools/gram_probe.py --config cfg4 --subjects 16 --finalize > $O/ncu.log 2>&1
SRM_B200_OZW=records timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_rowgemm" -s 2 -c 1 -f -o $O/rec_cfg4 \
   python tools/gram_probe.py --config cfg4 --subjects 16 --finalize > $O/ncu_rec.log 2>&1
