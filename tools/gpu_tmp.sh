# scratch: scaling/tweet timing for variants (2 rounds)
set -x
for r in 1 2; do for c in scaling tweet; do
  for v in ${VARIANTS}; do echo "== $v $c"; WMD_LIB=$v timeout 300 python tools/pass_timing.py $c auto 5; done
done; done
