# bench line + ncu launch list
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
python bench.py --config many --steps 2 --warmup 2 > gpurun_out/bench_many.json 2> gpurun_out/bench_many.err; echo many=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
