python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/r1_bench_config2.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/r1_bench_config2_reference.json 2>> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_bench_config2.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/launch_c2.log 2>&1
tail -c 300 gpurun_out/r1_bench_config2.json
