# scratch: build-kernel parity + timing (variants)
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "build or tiny or tweet or query_width or cta" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in tweet scaling long many; do
  echo "== main $c"; timeout 300 python tools/pass_timing.py $c auto 5
  for v in ${VARIANTS}; do echo "== $v $c"; WMD_LIB=$v timeout 300 python tools/pass_timing.py $c auto 5; done
done
