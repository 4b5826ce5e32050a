# round 2: multi-process (world 2 on one GPU, gloo) checks of the sharded path + bench N=2 code path
python -m pytest tests/test_dist_gpu.py tests/test_prox_gpu.py -q -x -m gpu -k "not C4" > gpurun_out/dist.log 2>&1; echo EXIT $? >> gpurun_out/dist.log
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config C3 --mode prox --steps 1 --warmup 3 --no-cpu --iters 100 > gpurun_out/b2p.json 2> gpurun_out/b2p.err; echo EXIT $? >> gpurun_out/b2p.err
