# round 2 (third pass): narrow strips (k_wave_n, 64-column k_wave_prox) -- tests then A/B bench lines
set -u
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py -k "narrow or strip_width or wave_edge or random_pass or C3" > gpurun_out/n_tests1.log 2>&1; echo "EXIT $?" >> gpurun_out/n_tests1.log
timeout 1500 python -m pytest -x -q tests/test_prox_wave_gpu.py > gpurun_out/n_tests2.log 2>&1; echo "EXIT $?" >> gpurun_out/n_tests2.log
tail -3 gpurun_out/n_tests1.log gpurun_out/n_tests2.log
B="python bench.py --no-cpu --steps 3 --warmup 3"
$B --config C3 > gpurun_out/n_C3.json 2> gpurun_out/n_C3.err
UOT_WAVE_V=4 $B --config C3 > gpurun_out/n_C3_v4.json 2> gpurun_out/n_C3_v4.err
$B --mode prox > gpurun_out/n_C4p.json 2> gpurun_out/n_C4p.err
UOT_PROX_W=16 $B --mode prox > gpurun_out/n_C4p_w16.json 2> gpurun_out/n_C4p_w16.err
UOT_PROX_V=4 $B --mode prox > gpurun_out/n_C4p_v4.json 2> gpurun_out/n_C4p_v4.err
UOT_PROX_PASS=3 $B --mode prox > gpurun_out/n_C4p_p3.json 2> gpurun_out/n_C4p_p3.err
UOT_PROX_WAVE=2 $B --config C3 --mode prox > gpurun_out/n_C3p.json 2> gpurun_out/n_C3p.err
$B --config C3 --mode prox > gpurun_out/n_C3p_auto.json 2> gpurun_out/n_C3p_auto.err
for f in gpurun_out/n_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r.get('kernels_in_step'), d['clocks'])" 2>&1 | tail -1; done
