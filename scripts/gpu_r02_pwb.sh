# chain-prox bench only (C4, C3)
UOT_DEBUG=1 timeout 300 python bench.py --mode prox --no-cpu --no-e2e > gpurun_out/pw_C4.json 2> gpurun_out/pw_C4.err
UOT_DEBUG=1 timeout 300 python bench.py --config C3 --mode prox --no-cpu --no-e2e > gpurun_out/pw_C3.json 2> gpurun_out/pw_C3.err
timeout 300 python -m pytest tests/test_prox_wave_gpu.py -q -x > gpurun_out/pw_tests.log 2>&1; tail -2 gpurun_out/pw_tests.log
for f in gpurun_out/pw_C*.json; do echo $f; grep plan ${f%.json}.err | head -1; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['kernels_in_step'])"; done
