set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python tools/pass_timing.py scaling fused 3 > gpurun_out/pt_scaling.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_fused -s 2 -c 2 -o gpurun_out/prof_fused python tools/pass_timing.py scaling fused 1 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
