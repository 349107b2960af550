# scratch: full tests + bench lines
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for c in scaling long tweet; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '%.4e'%d['value'], d['ms_per_step'], 'e2e %.4e'%d['e2e']['value'], (d.get('roofline') or {}).get('frac'), d.get('phases_ms_per_step'))"; done
timeout 300 python bench.py --config many --steps 2 --warmup 3 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('many qps', d['queries_per_s'], d['ms_per_step'])"
