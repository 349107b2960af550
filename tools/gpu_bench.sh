# bench lines of every config (round R, default r02): scaling (default build + path), scaling on
# the per-iteration path, long, many, tweet, tiny, and the reference arm; run ON the GPU box
R=${1:-r02}
set -x
mkdir -p gpurun_out/bench
python bench.py > gpurun_out/bench/${R}_bench_scaling.json 2> gpurun_out/bench/scaling.err; echo bench=$?
python bench.py --path iter --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench/${R}_bench_scaling_iter.json 2> gpurun_out/bench/iter.err; echo iter=$?
for c in long many tweet tiny; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench/${R}_bench_$c.json 2> gpurun_out/bench/$c.err; echo $c=$?
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench/${R}_bench_reference.json 2> gpurun_out/bench/ref.err; echo ref=$?
tail -n1 gpurun_out/bench/*.json | cut -c1-300
