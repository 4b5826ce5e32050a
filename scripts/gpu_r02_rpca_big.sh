# round 2: Algorithm 3 beyond 128 frames (subspace SVT), and the RPCA regressions
python -m pytest tests/test_rpca_big_gpu.py tests/test_rpca_gpu.py tests/test_rpca_shard_gpu.py -q -x -m gpu > gpurun_out/rpca_big.log 2>&1; echo EXIT $? >> gpurun_out/rpca_big.log
