# scratch: full GPU tests + Long/Scaling timing
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for c in long scaling tweet; do timeout 300 python tools/pass_timing.py $c auto 5; done
