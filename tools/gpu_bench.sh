# bench lines (scaling, long, many, reference arm) + ncu launch list of the default bench command
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.json
python bench.py --config long --steps 5 --warmup 3 > gpurun_out/bench_long.json 2> gpurun_out/bench_long.err; echo long=$?
tail -1 gpurun_out/bench_long.json
python bench.py --config many --steps 2 --warmup 3 > gpurun_out/bench_many.json 2> gpurun_out/bench_many.err; echo many=$?
tail -1 gpurun_out/bench_many.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
python bench.py --config long --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_long_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_long.csv \
  python bench.py --config long --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_long.log 2>&1; echo ncu_long=$?
