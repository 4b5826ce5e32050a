# RPCA T > 128: pipelined Gram blocks -- RPCA GPU tests, C4-video stage timings with / without
set -u
timeout 1500 python -m pytest -x -q tests/test_rpca_big_gpu.py tests/test_rpca_shard_gpu.py tests/test_rpca_gpu.py > gpurun_out/gp_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gp_tests.log
tail -2 gpurun_out/gp_tests.log
python scripts/bench_rpca.py 20 1 C4 > gpurun_out/gp_c4.json 2>/dev/null
UOT_RPCA_GRAM_PIPE=0 python scripts/bench_rpca.py 20 1 C4 > gpurun_out/gp_c4_old.json 2>/dev/null
for f in gp_c4 gp_c4_old; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['us_per_iter'], d['stage_us_per_iter'], d['report']['objective'])"; done
