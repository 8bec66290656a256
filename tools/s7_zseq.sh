# session 7: final W with both feature halves of an item on one CTA (SRM_B200_OZW_ZSEQ) -- parity, A/B on cfg 3 / cfg 5 / cfg 2(K=50: unaffected)
set -x
O=gpurun_out/s7z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "final_w or fp32_configs or int8_gram_fit" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in cfg3 cfg5; do for z in 0 1 0 1; do
  SRM_B200_OZW_ZSEQ=$z timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
     > $O/${c}_z${z}_$RANDOM.json 2> $O/${c}_z$z.err
done; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/s7z/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d['roofline_hbm']['kernels']['oz_w']
        print(f, 'step %.2f ms' % d['ms_per_step'], 'oz_w %.2f ms frac %.3f' % (k['ms'], k['frac']))
    except Exception as e:
        print(f, 'ERR', e)
PY
tail -3 $O/pytest.log
