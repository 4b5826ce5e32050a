# chain-prox wavefront (k_wave_prox): parity tests + C3 / C4 chain-prox bench
set -u
timeout 900 python -m pytest tests/test_prox_wave_gpu.py -q > gpurun_out/pw_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/pw_tests.log
timeout 900 python -m pytest tests/test_prox_gpu.py tests/test_dist_gpu.py -x -q -k "not C4" > gpurun_out/pw_tests2.log 2>&1; echo "EXIT $?" >> gpurun_out/pw_tests2.log
timeout 900 python scripts/dev/pw_debug.py > gpurun_out/pw_debug.log 2>&1
UOT_DEBUG=1 timeout 300 python bench.py --mode prox --no-cpu --no-e2e > gpurun_out/pw_C4.json 2> gpurun_out/pw_C4.err
UOT_DEBUG=1 UOT_PROX_CL=8 timeout 300 python bench.py --mode prox --no-cpu --no-e2e > gpurun_out/pw8_C4.json 2> gpurun_out/pw8_C4.err
UOT_DEBUG=1 timeout 300 python bench.py --config C3 --mode prox --no-cpu --no-e2e > gpurun_out/pw_C3.json 2> gpurun_out/pw_C3.err
tail -n 5 gpurun_out/pw_tests.log gpurun_out/pw_tests2.log
for f in gpurun_out/pw*_C*.json; do echo $f; grep plan ${f%.json}.err | head -2; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['kernels_in_step'])"; done
