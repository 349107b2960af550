python -m paper_2005_06727_b200.build > /dev/null 2>&1
python tools/pass_timing.py long auto 1 > gpurun_out/plain_fb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fallback -s 2 -c 1 -o gpurun_out/prof_fallback python tools/pass_timing.py long auto 1 > gpurun_out/ncu_fb.log 2>&1; echo ncu=$?
