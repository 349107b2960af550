python -m paper_2005_06727_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for c in scaling tweet many; do echo "== D2 $c"; python tools/pass_timing.py $c auto 5; echo "== D1 $c"; WMD_LIB=variants/lib_d1.so python tools/pass_timing.py $c auto 5; done
