#!/bin/bash
# Runs on the GPU box (gpurun): ncu launch list of the default bench command plus one full capture of every hot
# kernel at the sizes DESIGN.md quotes.  Writes raw reports to gpurun_out/ and text summaries to profiles/.
set -u
R=${1:-r2}
mkdir -p gpurun_out profiles
NCU="ncu --set full --clock-control none --import-source on"
# launch list of the bench command (cold-cache, serialised: shares, not absolutes, are comparable)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file profiles/${R}_launches_bench_config2.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/launch_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file profiles/${R}_launches_bench_config3.csv \
    python bench.py --workload config3 --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/launch_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file profiles/${R}_launches_bench_config4.csv \
    python bench.py --workload config4_fixed --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/launch_c4.log 2>&1
cap() {  # name kernel-regex skip units unit-name -- target args
  local name=$1 rx=$2 skip=$3 units=$4 uname=$5; shift 5
  $NCU -k regex:$rx -s $skip -c 1 -o gpurun_out/${R}_$name -f python scripts/profile_target.py "$@" > gpurun_out/cap_$name.log 2>&1
  { echo "# ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1; workload: scripts/profile_target.py $*";
    python scripts/ncu_summary.py gpurun_out/${R}_$name.ncu-rep $units $uname; } > profiles/${R}_ncu_$name.txt 2>/dev/null
  rm -f gpurun_out/${R}_$name.ncu-rep   # the text summary is what is kept (gpurun_out/ is capped at 64 MiB)
}
cap vsample_config2 vsample 2 32768 warp-sample vsample f2 6 1e6
cap reduce_config2 reduce_kernel 5 1 launch run f2 6 1e6
cap finish_config2 finish_kernel 5 1 launch run f2 6 1e6
cap vsample_config4 vsample 1 26873856 warp-sample vsample f3 8 1e9
cap pagani_lanes_f1_d8 pagani_eval 2 390625 region eval f1 8 5
cap pagani_lanes_f4_d8 pagani_eval 2 390625 region eval f4 8 5
cap pagani_lanes_f2_d8 pagani_eval 2 390625 region eval f2 8 5
cap pagani_lanes_f3_d8 pagani_eval 2 390625 region eval f3 8 5
cap pagani_warp_f4_d5_small pagani_eval 2 1024 region eval f4 5 4
cap pagani_warp_f1_d8_small pagani_eval 2 6561 region eval f1 8 3
# the final bench lines (own arm with the secondary workloads, reference arm) and the config-5 sweep
python bench.py > profiles/${R}_bench_config2.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > profiles/${R}_bench_config2_reference.json 2>> gpurun_out/bench_final.err
python scripts/sweep.py --out profiles/${R}_sweep_config5 > gpurun_out/sweep.log 2>&1
for fam in f1 f2 f3 f4 f5 f6; do python scripts/eval_bench.py $fam 8 6; done > profiles/${R}_eval_bench.txt 2>&1
python scripts/refine_bench.py > profiles/${R}_refine_bench.txt 2>&1
{ echo "# PCB_NO_PDL=1 PCB_PAGANI_PUBLISH=0: plain launches, scalars by copy + synchronise"; PCB_NO_PDL=1 PCB_PAGANI_PUBLISH=0 python scripts/refine_bench.py; } >> profiles/${R}_refine_bench.txt 2>&1
timeout 120 scripts/micro/atom > profiles/${R}_micro_shared_atomics.txt 2>&1
python scripts/cold_call.py > profiles/${R}_cold_call.txt 2>&1
ls -la profiles/
# device timeline of one config-2 run (%globaltimer stamps per kernel and phase; PCB_TIMELINE=1)
python scripts/timeline_run.py f2 6 1e6 2>&1 | tail -50 > profiles/${R}_timeline_config2.txt
python scripts/timeline_run.py f3 8 1e9 2>&1 | tail -50 > profiles/${R}_timeline_config4.txt
