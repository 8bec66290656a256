# session 7: the time guard of tests/test_gpu_baseline.py -- forced slices (tiny budget), then the file at its defaults
set -x
O=gpurun_out/s7guard
mkdir -p $O
SRM_GPU_SUITE_BUDGET_S=150 SRM_PARITY_REPORT=$O/sliced timeout 900 python -m pytest tests/test_gpu_baseline.py -q -m gpu -x -W default -k "cfg3 or cfg4 or cfg5" > $O/sliced.log 2>&1; echo "rc=$?" >> $O/sliced.log
tail -n 15 $O/sliced.log
SRM_PARITY_REPORT=$O/full timeout 1500 python -m pytest tests/test_gpu_baseline.py -q -m gpu -x -W default --durations=8 > $O/full.log 2>&1; echo "rc=$?" >> $O/full.log
tail -n 20 $O/full.log
