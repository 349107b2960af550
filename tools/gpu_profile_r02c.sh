#!/bin/bash
# Round-2 (third pass: FFMA2 kernels, load_D fix) ncu captures, run ON the GPU box from the repo root (gpurun), after the
# exact tensor-core build and the half-warp fused kernel: full-set captures of one Scaling query's
# fused launches (half-warp kernel, 6 length buckets) and distance build, of one Long query's
# one-CTA launches, summarised on the box into gpurun_out/prof/ (the .ncu-rep files stay in /tmp:
# they exceed gpurun's copy-back cap), plus the launch list of a whole bench run. Each capture runs
# after its command exited 0 alone.
set -u
mkdir -p gpurun_out/prof
R=/tmp/ncu_r02c; rm -rf $R; mkdir -p $R   # a reused box keeps /tmp: never summarise an old report
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench"
$B > gpurun_out/prof/plain_scaling.log 2>&1 || exit 3
ncu -f --set full --import-source on --clock-control none -k regex:"sinkhorn_half" --launch-skip 6 --launch-count 6 \
    -o $R/scaling_half $B > gpurun_out/prof/ncu_scaling_half.log 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:"build_mx" --launch-skip 1 --launch-count 1 \
    -o $R/scaling_build $B > gpurun_out/prof/ncu_scaling_build.log 2>&1
$B --config long > gpurun_out/prof/plain_long.log 2>&1 || exit 4
ncu -f --set full --import-source on --clock-control none -k regex:"sinkhorn_cta" --launch-skip 8 --launch-count 8 \
    -o $R/long_cta $B --config long > gpurun_out/prof/ncu_long_cta.log 2>&1
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_scaling.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-roofbench > gpurun_out/prof/ncu_launches.log 2>&1
for r in scaling_half scaling_build long_cta; do
  [ -f $R/$r.ncu-rep ] || continue
  python tools/ncu_summary.py $R/$r.ncu-rep --raw --stalls > gpurun_out/prof/${r}_summary.txt 2>&1
done
python tools/ncu_source.py $R/scaling_half.ncu-rep "(int)8, (int)2, (int)0" --top 50 > gpurun_out/prof/scaling_half_source_hot.txt 2>&1
python tools/ncu_source.py $R/long_cta.ncu-rep "(int)13, (int)8, (int)0" --top 50 > gpurun_out/prof/long_cta_source_hot.txt 2>&1
python tools/ncu_source.py $R/scaling_build.ncu-rep "build_mx_exact" --top 40 > gpurun_out/prof/scaling_build_source_hot.txt 2>&1
python tools/ncu_traffic.py $R/scaling_half.ncu-rep scaling sinkhorn_half gpurun_out/prof/r02_traffic.json
python tools/ncu_traffic.py $R/long_cta.ncu-rep long sinkhorn_cta gpurun_out/prof/r02_traffic.json
python tools/ncu_traffic.py $R/scaling_build.ncu-rep scaling_build build_mx_exact gpurun_out/prof/r02_traffic.json
ls -la $R gpurun_out/prof
