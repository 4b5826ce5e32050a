# Algorithm 3: threshold-Jacobi round skipping in k_rp_eig -- RPCA GPU tests, then C3-video stage
# timings with and without (UOT_RPCA_EIG_SKIP=0)
set -u
timeout 1500 python -m pytest -x -q tests/test_rpca_gpu.py tests/test_rpca_shard_gpu.py tests/test_rpca_big_gpu.py > gpurun_out/rs_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/rs_tests.log
tail -3 gpurun_out/rs_tests.log
UOT_RPCA_DEBUG=1 python scripts/bench_rpca.py 200 > gpurun_out/rs_skip.json 2> gpurun_out/rs_skip.err
UOT_RPCA_DEBUG=1 UOT_RPCA_EIG_SKIP=0 python scripts/bench_rpca.py 200 > gpurun_out/rs_noskip.json 2> gpurun_out/rs_noskip.err
for f in rs_skip rs_noskip; do echo $f; tail -1 gpurun_out/$f.err; python -c "import json; d=json.load(open('gpurun_out/$f.json')); print(d['us_per_iter'], d['stage_us_per_iter'], d['report']['objective'], d['report']['jacobi_sweeps'])"; done
