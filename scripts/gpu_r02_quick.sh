timeout 1200 python -m pytest tests/test_dist_gpu.py -q -x -m gpu -k "bench" > gpurun_out/quick.log 2>&1; echo EXIT $? >> gpurun_out/quick.log
