# chain-prox wavefront: tests (prox, dist, wave, variants, parity) + C4/C3 prox bench
set -u
timeout 1500 python -m pytest tests/test_prox_wave_gpu.py tests/test_prox_gpu.py tests/test_dist_gpu.py tests/test_variants_gpu.py -q -k "not C4_full" > gpurun_out/pwt_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/pwt_tests.log
tail -4 gpurun_out/pwt_tests.log
bash scripts/gpu_r02_pwb.sh
