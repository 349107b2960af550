#!/bin/bash
# Round-2 ncu captures, run ON the GPU box from the repo root (gpurun): full-set captures of the
# Scaling fused-phase launches + distance build, and of the Long one-CTA launches, summarised on
# the box into gpurun_out/ (the .ncu-rep files stay in /tmp: they exceed gpurun's copy-back cap),
# plus the launch list of a whole bench run. Each capture runs after its command exited 0 alone.
set -u
mkdir -p gpurun_out/prof
R=/tmp/ncu_r02; mkdir -p $R
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench > gpurun_out/prof/plain_scaling.log 2>&1 || exit 3
ncu --set full --import-source on --clock-control none -k regex:"sinkhorn_fused" --launch-skip 3 --launch-count 3 \
    -o $R/scaling_fused python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench > gpurun_out/prof/ncu_scaling_fused.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"build_mx" --launch-skip 1 --launch-count 1 \
    -o $R/scaling_build python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench > gpurun_out/prof/ncu_scaling_build.log 2>&1
python bench.py --config long --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench > gpurun_out/prof/plain_long.log 2>&1 || exit 4
ncu --set full --import-source on --clock-control none -k regex:"sinkhorn_cta" --launch-skip 5 --launch-count 5 \
    -o $R/long_cta python bench.py --config long --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench > gpurun_out/prof/ncu_long_cta.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_scaling.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-roofbench > gpurun_out/prof/ncu_launches.log 2>&1
for r in scaling_fused scaling_build long_cta; do
  [ -f $R/$r.ncu-rep ] || continue
  python tools/ncu_summary.py $R/$r.ncu-rep --raw --stalls > gpurun_out/prof/${r}_summary.txt 2>&1
done
python tools/ncu_source.py $R/scaling_fused.ncu-rep "(int)4, (int)1, (int)0" --top 50 > gpurun_out/prof/scaling_fused_source_hot.txt 2>&1
python tools/ncu_source.py $R/long_cta.ncu-rep "sinkhorn_cta_kernel" --top 50 > gpurun_out/prof/long_cta_source_hot.txt 2>&1
python tools/ncu_traffic.py $R/scaling_fused.ncu-rep scaling sinkhorn_fused gpurun_out/prof/r02_traffic.json
python tools/ncu_traffic.py $R/long_cta.ncu-rep long sinkhorn_cta gpurun_out/prof/r02_traffic.json
ls -la $R gpurun_out/prof
