for l in libparcube_b200.so libpcb_old.so; do echo == $l; for cfg in "f3 8 1e9" "f2 6 1e6" "f3 6 1e9" "f3 5 1e9"; do PCB_LIB_NAME=$l python scripts/pass_bench.py $cfg 5; done; done
python scripts/timeline_run.py f2 6 1e6 2>&1 | grep "CTA 0 batch\|it 1 vsample\|device sec" | tail -16
python bench.py --workload config4 --steps 3 --warmup 3 --no-extras --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config4', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
python bench.py --no-extras --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config2', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['avg_launch_ms'])"
