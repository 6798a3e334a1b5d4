python -m pytest tests/test_gpu_mcubes.py tests/test_gpu_sharded.py tests/test_gpu_cli.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
python bench.py --no-extras --no-cpu-baseline > gpurun_out/ev_off.json 2> gpurun_out/pdl_on.err
PCB_MC_ITER_EVENTS=1 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ev_on.json 2> gpurun_out/pdl_off.err
PCB_NO_PDL=1 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ev_off_nopdl.json 2> gpurun_out/pdl_off.err
python - <<'P'
import json
for f in ['ev_off','ev_on','ev_off_nopdl']:
    d=json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1])
    print(f, d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['ms_per_step_with_event_pairs'])
P
done
