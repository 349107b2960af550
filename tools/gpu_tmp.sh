# scratch: CTA tests + Long timing
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "cta or long or auto_path or grid or width or single or build" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in long; do timeout 300 python tools/pass_timing.py $c auto 5; done
