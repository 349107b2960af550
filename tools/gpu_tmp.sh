# scratch: full GPU tests + timing of all configs + many bench
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for c in tweet many scaling long; do timeout 300 python tools/pass_timing.py $c auto 5; done
timeout 300 python bench.py --config many --steps 2 --warmup 3 --no-cpu-baseline | tail -1 | cut -c1-400
