# session 7: k_oz_split_f32 walking groups of voxel blocks (SRM_B200_SPLIT_F32_GROUPS) -- parity, then sweep on cfg 4 / cfg 3
set -x
O=gpurun_out/s7
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "fp32 or extreme or int8_gram_matches" > $O/pytest_fp32.log 2>&1; echo "rc=$?" >> $O/pytest_fp32.log
for nb in 4 2; do for g in 1 2 4 8 16; do
  SRM_B200_SPLIT_NB=$nb SRM_B200_SPLIT_F32_GROUPS=$g timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
     > $O/cfg4_nb${nb}_g$g.json 2> $O/cfg4_nb${nb}_g$g.err
done; done
for g in 1 4 8; do
  SRM_B200_SPLIT_F32_GROUPS=$g timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
     > $O/cfg3_nb4_g$g.json 2> $O/cfg3_nb4_g$g.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/s7/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d['roofline_hbm']['kernels']['oz_split']
        print(f, 'step %.2f ms' % d['ms_per_step'], 'split %.2f ms frac %.3f' % (k['ms'], k['frac']))
    except Exception as e:
        print(f, 'ERR', e)
PY
