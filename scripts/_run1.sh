python -m pytest tests/test_gpu_pagani.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
for f in f1 f4 f5 f6; do for dg in "8 5" "7 6" "6 8" "5 16"; do python scripts/eval_bench.py $f $dg 5 2>&1 | grep -i lanes; done; done
python bench.py --workload config3 --no-extras --no-cpu-baseline --steps 3 --warmup 3 | cut -c1-200
