# round 2: sharded Algorithm 3 (emulated shards + world-2 processes) and the RPCA regressions
python -m pytest tests/test_rpca_shard_gpu.py tests/test_rpca_gpu.py tests/test_dist_gpu.py -q -m gpu > gpurun_out/rpca_shard.log 2>&1; echo EXIT $? >> gpurun_out/rpca_shard.log
