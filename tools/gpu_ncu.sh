# ncu --set full of the fused kernels on one config (args: CONFIG, KREGEX, COUNT)
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
C=${CONFIG:-scaling}; K=${KREGEX:-sinkhorn_fused}; N=${COUNT:-4}
python tools/pass_timing.py $C auto 1 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-8} -c $N -o gpurun_out/prof_${TAG:-x} python tools/pass_timing.py $C auto 1 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_full.log
