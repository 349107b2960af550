# one GPU round-trip: build, parity tests, phase timing (args: configs for pass_timing)
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-tiny tweet many scaling}; do timeout 300 python tools/pass_timing.py $c auto 5; done > gpurun_out/pt.log 2>&1
cat gpurun_out/pt.log
