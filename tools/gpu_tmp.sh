# scratch: full GPU tests + timing of all configs (main, variants)
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
WMD_LIB=variants/libwmd_big12.so timeout 900 python -m pytest tests -m gpu -q -k "cta or long" > gpurun_out/pytest_gpu_v.log 2>&1; echo pytest_v=$?
tail -2 gpurun_out/pytest_gpu_v.log
for c in long; do
  echo "== main $c"; timeout 300 python tools/pass_timing.py $c auto 5
  for v in ${VARIANTS}; do echo "== $v $c"; WMD_LIB=$v timeout 300 python tools/pass_timing.py $c auto 5; done
done
