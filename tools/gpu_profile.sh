# round-end profiles: ncu --set full of the fused phase (Scaling: one query's 3 bucket launches;
# Long: 5 CTA launches) and of the distance build, summarised on the box (the reports are large);
# then the launch lists of the bench commands
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
rm -rf /tmp/reps; mkdir -p /tmp/reps gpurun_out/prof
python tools/pass_timing.py scaling auto 1 > gpurun_out/prof/plain_scaling.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:sinkhorn_fused -s 6 -c 3 -o /tmp/reps/r01_full_scaling_fused python tools/pass_timing.py scaling auto 1 > gpurun_out/prof/ncu1.log 2>&1; echo ncu1=$?
python tools/pass_timing.py long auto 1 > gpurun_out/prof/plain_long.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:sinkhorn_cta -s 10 -c 5 -o /tmp/reps/r01_full_long_cta python tools/pass_timing.py long auto 1 > gpurun_out/prof/ncu2.log 2>&1; echo ncu2=$?
ncu -f --set full --clock-control none --import-source on -k regex:build_mx_tc -s 2 -c 1 -o /tmp/reps/r01_full_scaling_build python tools/pass_timing.py scaling auto 1 > gpurun_out/prof/ncu3.log 2>&1; echo ncu3=$?
for r in r01_full_scaling_fused r01_full_long_cta r01_full_scaling_build; do
  python tools/ncu_summary.py /tmp/reps/$r.ncu-rep --raw > gpurun_out/prof/${r}_summary.txt 2>&1
done
python tools/ncu_source.py /tmp/reps/r01_full_scaling_fused.ncu-rep "(int)1, (int)0" --top 40 > gpurun_out/prof/r01_full_scaling_fused_source_hot.txt 2>&1
python tools/ncu_source.py /tmp/reps/r01_full_long_cta.ncu-rep "(int)8, (int)0" --top 40 > gpurun_out/prof/r01_full_long_cta_source_hot.txt 2>&1
python tools/ncu_traffic.py /tmp/reps/r01_full_scaling_fused.ncu-rep scaling sinkhorn_fused gpurun_out/prof/r01_traffic.json
python tools/ncu_traffic.py /tmp/reps/r01_full_long_cta.ncu-rep long sinkhorn_cta gpurun_out/prof/r01_traffic.json
cp /tmp/reps/r01_full_scaling_build.ncu-rep gpurun_out/prof/ 2>/dev/null
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/prof/r01_launches_scaling.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_l1.log 2>&1; echo ncu_l1=$?
python bench.py --config long --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_long_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/prof/r01_launches_long.csv \
  python bench.py --config long --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_l2.log 2>&1; echo ncu_l2=$?
du -sh gpurun_out/prof
