mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2/smi.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s2/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s2/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/quick.sh s2
