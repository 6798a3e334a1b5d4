python -m pytest tests/test_gpu_mcubes.py tests/test_gpu_sharded.py tests/test_gpu_cli.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do python bench.py --no-extras --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config2', d['ms_per_step'], d['e2e']['ms_per_step'], d['result'])"; done
