python -m pytest tests/test_gpu_pagani.py tests/test_gpu_sharded.py tests/test_gpu_cli.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
python bench.py --workload config1 --steps 200 --warmup 20 --no-extras --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config1', d['ms_per_step'], d['e2e']['ms_per_step'], d['result'])"
PCB_NO_PDL=1 python bench.py --workload config1 --steps 200 --warmup 20 --no-extras --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config1 nopdl', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
