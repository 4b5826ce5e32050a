# round 2: k_single (one-CTA kernel for single small pairs) + regressions of the forced-path tests + C1 bench
python -m pytest tests/test_single_gpu.py tests/test_parity_gpu.py tests/test_variants_gpu.py -q -x -m gpu > gpurun_out/single.log 2>&1; echo EXIT $? >> gpurun_out/single.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT $? >> gpurun_out/smoke.log
python bench.py --config C1 --steps 5 --warmup 3 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo EXIT $? >> gpurun_out/b_c1.err
