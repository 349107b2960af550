# scratch: build parity for variants + timing
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
for v in ${VARIANTS}; do WMD_LIB=$v timeout 900 python -m pytest tests -m gpu -x -q -k "build or tiny or tweet or width" 2>&1 | tail -1; done
for c in many long tweet; do
  echo "== main $c"; timeout 300 python tools/pass_timing.py $c auto 5
  for v in ${VARIANTS}; do echo "== $v $c"; WMD_LIB=$v timeout 300 python tools/pass_timing.py $c auto 5; done
done
