# time the fused phase of several library variants (VARIANTS="a.so b.so", CONFIGS)
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
for c in ${CONFIGS:-scaling}; do
  echo "== main $c"; python tools/pass_timing.py $c auto 5
  for v in ${VARIANTS}; do echo "== $v $c"; WMD_LIB=$v python tools/pass_timing.py $c auto 5; done
done
