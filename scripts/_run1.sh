python -m pytest tests/test_gpu_pagani.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
for lib in libpcb_base.so libparcube_b200.so; do
export PCB_LIB_NAME=$lib
echo "== $lib"
for f in f1 f2 f4; do for dg in "8 5" "7 6" "6 8" "5 16"; do python scripts/eval_bench.py $f $dg 5 2>&1 | grep -i lanes; done; done
for dg in "9 4" "10 3"; do python scripts/eval_bench.py f1 $dg 3 2>&1 | grep -i "lanes\|warp"; python scripts/eval_bench.py f4 $dg 3 2>&1 | grep -i "lanes\|warp"; done
python bench.py --workload config3 --no-extras --no-cpu-baseline --steps 3 --warmup 3 | cut -c1-200
done
