# session 7: full ncu captures of the fp32 one-time kernels at HEAD (cfg 4 shape, 16 subjects): four-slice Gram, fp32 slicing, final W at kp = 64 and kp = 128 (zseq)
set -x
O=gpurun_out/s7ncu
mkdir -p $O
timeout 600 python tools/gram_probe.py --config cfg4 --subjects 16 --finalize > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gram" -s 1 -c 1 \
   -f -o $O/oz_gram4_cfg4 python tools/gram_probe.py --config cfg4 --subjects 16 > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_split_f32" -s 1 -c 1 \
   -f -o $O/oz_split_f32_cfg4 python tools/gram_probe.py --config cfg4 --subjects 16 > $O/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_rowgemm" -c 1 \
   -f -o $O/ozw_cfg4 python bench.py --config cfg4 --subjects 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_rowgemm" -c 1 \
   -f -o $O/ozw_cfg5_zseq python bench.py --config cfg5 --subjects 16 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu4.log 2>&1
ls -la $O
