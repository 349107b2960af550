python -m paper_2005_06727_b200.build > /dev/null 2>&1
for c in tiny tweet; do
python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'direct', d['ms_per_step'], d['e2e']['value'])"
python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --graph 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'graph', d['ms_per_step'], d['e2e']['value'])"
done
timeout 300 python -m pytest tests -m gpu -x -q -k graph 2>&1 | tail -1
