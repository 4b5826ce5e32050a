python bench.py > gpurun_out/r02c_bench_C4.json 2> gpurun_out/r02c_bench_C4.err; echo "EXIT $?" >> gpurun_out/r02c_bench_C4.err
bash scripts/gpu_r02_alltests.sh
