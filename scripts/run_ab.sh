python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/r1_bench_config2.json 2> gpurun_out/bench_final.err; tail -3 gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/r1_bench_config2_reference.json 2>> gpurun_out/bench_final.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/r1_bench_config2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])
for k,v in d['other_workloads'].items(): print(k, v['time_to_epsrel_s'], v['e2e_evals_per_s'], v['roofline_frac'])
P
