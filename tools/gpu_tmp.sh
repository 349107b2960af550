# scratch: full GPU tests, timing, shard projection
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
for c in scaling long tweet many; do timeout 300 python tools/pass_timing.py $c auto 5; done
python tools/shard_projection.py scaling 1 8 2>&1 | tail -2 | cut -c1-200
