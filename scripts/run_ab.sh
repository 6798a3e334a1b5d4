R=r1
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  local name=$1 rx=$2 skip=$3 units=$4 uname=$5; shift 5
  $NCU -k regex:$rx -s $skip -c 1 -o gpurun_out/${R}_$name -f python scripts/profile_target.py "$@" > gpurun_out/cap_$name.log 2>&1
  { echo "# ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1; workload: scripts/profile_target.py $*";
    python scripts/ncu_summary.py gpurun_out/${R}_$name.ncu-rep $units $uname; } > gpurun_out/${R}_ncu_$name.txt 2>/dev/null
}
cap reduce_config2 reduce_kernel 5 1 launch run f2 6 1e6
cap finish_config2 finish_kernel 5 1 launch run f2 6 1e6
head -14 gpurun_out/r1_ncu_reduce_config2.txt gpurun_out/r1_ncu_finish_config2.txt
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 600 gpurun_out/final_bench.json
