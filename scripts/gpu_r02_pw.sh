# chain prox: wave + ghost-pair tests, the world-2/3 drivers and the two-rank bench
timeout 1500 python -m pytest tests/test_prox_wave_gpu.py tests/test_dist_gpu.py tests/test_abi.py tests/test_prox_gpu.py -q > gpurun_out/pw_tests.log 2>&1; tail -3 gpurun_out/pw_tests.log
grep -E "^E |^FAILED" gpurun_out/pw_tests.log | head -20
timeout 300 python bench.py --mode prox --no-cpu --no-e2e > gpurun_out/pw_C4.json 2> gpurun_out/pw_C4.err
python -c "import json; d=json.loads(open('gpurun_out/pw_C4.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['kernels_in_step'])"
