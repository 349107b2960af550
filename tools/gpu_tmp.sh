# scratch: full GPU tests, fault-shape repros, timing
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
export NOFB=1
for spec in "44 257" "44 262" "41 270" "100 70" "128 70" "48 300"; do set -- $spec
  r=$(timeout 60 python tools/cta_repro.py $1 $2 2>&1 | tail -1 | cut -c1-60); echo "== v=$1 n=$2: $r"; done
unset NOFB
for c in scaling long tweet many; do timeout 300 python tools/pass_timing.py $c auto 5; done
