# the full GPU suite (what the driver runs at round end) + smoke
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
tail -5 gpurun_out/gpu_all.log; tail -6 gpurun_out/smoke.log
