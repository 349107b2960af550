# round-end bench lines: scaling (default), long, many, tweet, tiny, and the reference arm
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/bench
python bench.py > gpurun_out/bench/r01_bench_scaling.json 2> gpurun_out/bench/scaling.err; echo bench=$?
for c in long many tweet tiny; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench/r01_bench_$c.json 2> gpurun_out/bench/$c.err; echo $c=$?
done
python bench.py --graph --config tiny --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench/r01_bench_tiny_graph.json 2> gpurun_out/bench/tg.err; echo tg=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench/r01_bench_reference.json 2> gpurun_out/bench/ref.err; echo ref=$?
tail -n1 gpurun_out/bench/*.json | cut -c1-300
