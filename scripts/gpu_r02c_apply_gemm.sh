# RPCA T > 128: register-blocked apply GEMM -- RPCA GPU tests, then C4-video stage timings with and
# without it (UOT_RPCA_APPLY_GEMM=0: k_rp_apply_big)
set -u
timeout 1500 python -m pytest -x -q tests/test_rpca_big_gpu.py tests/test_rpca_shard_gpu.py tests/test_rpca_gpu.py > gpurun_out/ag_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/ag_tests.log
tail -2 gpurun_out/ag_tests.log
python scripts/bench_rpca.py 20 1 C4 > gpurun_out/ag_c4.json 2>/dev/null
UOT_RPCA_APPLY_GEMM=0 python scripts/bench_rpca.py 20 1 C4 > gpurun_out/ag_c4_old.json 2>/dev/null
for f in ag_c4 ag_c4_old; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['us_per_iter'], d['stage_us_per_iter'], d['report']['objective'])"; done
