# ncu --set full of the per-iteration pass kernel (CONFIG, TAG)
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
C=${CONFIG:-scaling}
python tools/pass_timing.py $C iter 1 > gpurun_out/ncu_plain_iter.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_pass -s ${SKIP:-45} -c ${COUNT:-2} -o gpurun_out/prof_${TAG:-iter} python tools/pass_timing.py $C iter 1 > gpurun_out/ncu_iter.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_iter.log
