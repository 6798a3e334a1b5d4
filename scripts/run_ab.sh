python -m pytest tests/test_gpu_mcubes.py tests/test_gpu_sharded.py tests/test_gpu_cli.py -m gpu -x -q 2>&1 | tail -15
python scripts/timeline_run.py f2 6 1e6 2>&1 | tail -36
python bench.py --no-extras --no-cpu-baseline > gpurun_out/opt.json 2> gpurun_out/opt.err
python - <<'P'
import json
for f in ['opt']:
    d=json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1])
    print(f, d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['ms_per_step_with_event_pairs'], d['result'])
P
