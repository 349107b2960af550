# scratch: timing main vs no-stream + DRAM traffic of the fused phase (ncu metrics only)
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
for r in 1 2; do
  echo "== main"; timeout 300 python tools/pass_timing.py scaling auto 5
  for v in ${VARIANTS}; do echo "== $v"; WMD_LIB=$v timeout 300 python tools/pass_timing.py scaling auto 5; done
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sinkhorn_fused -s 6 -c 3 --csv python tools/pass_timing.py scaling auto 1 2>/dev/null | grep -E "dram__bytes" | awk -F'","' '{print $(NF-2), $NF}' | head -6
echo "== nostream ncu"
WMD_LIB=variants/libwmd_nostream.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sinkhorn_fused -s 6 -c 3 --csv python tools/pass_timing.py scaling auto 1 2>/dev/null | grep -E "dram__bytes" | awk -F'","' '{print $(NF-2), $NF}' | head -6
