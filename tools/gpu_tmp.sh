# scratch: full GPU tests + timing
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
for c in scaling long; do timeout 300 python tools/pass_timing.py $c auto 5; done
