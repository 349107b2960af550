set -u
mkdir -p gpurun_out/prof
R=/tmp/ncu_half; rm -rf $R; mkdir -p $R
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-roofbench"
$B > gpurun_out/prof/plain_scaling.log 2>&1 || exit 3
ncu -f --set full --import-source on --clock-control none -k regex:"sinkhorn_half" --launch-skip 6 --launch-count 6 \
    -o $R/scaling_half $B > gpurun_out/prof/ncu_scaling_half.log 2>&1
python tools/ncu_summary.py $R/scaling_half.ncu-rep --raw --stalls > gpurun_out/prof/scaling_half_summary.txt 2>&1
python tools/ncu_source.py $R/scaling_half.ncu-rep "(int)8, (int)2, (int)0" --top 60 > gpurun_out/prof/scaling_half_source_hot.txt 2>&1
python tools/ncu_traffic.py $R/scaling_half.ncu-rep scaling sinkhorn_half gpurun_out/prof/traffic_half.json
