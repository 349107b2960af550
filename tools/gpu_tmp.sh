# scratch: CTA tests + long timing + DRAM traffic of the CTA phase
set -x
python -m paper_2005_06727_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "cta or long or reanchor" 2>&1 | tail -1
for r in 1 2; do timeout 300 python tools/pass_timing.py long auto 3; done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sinkhorn_cta -s 10 -c 5 --csv python tools/pass_timing.py long auto 1 2>/dev/null | grep -E "dram__bytes" | awk -F'","' '{print $(NF-2), $NF}' | head -10
