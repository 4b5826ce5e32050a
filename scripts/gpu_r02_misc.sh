timeout 900 python -m pytest tests/test_dist_gpu.py -q -x -m gpu > gpurun_out/dist2.log 2>&1; echo EXIT $? >> gpurun_out/dist2.log
timeout 300 python scripts/host_overhead.py > gpurun_out/host_overhead.json 2> gpurun_out/host_overhead.err
