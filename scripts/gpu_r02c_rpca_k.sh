# RPCA T > 128: subspace width k = 64 (documented default) vs 128 -- tests, C4 video timing + certificate
set -u
timeout 1500 python -m pytest -x -q tests/test_rpca_big_gpu.py tests/test_rpca_shard_gpu.py > gpurun_out/rk_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/rk_tests.log
grep -E "AssertionError|passed|failed" gpurun_out/rk_tests.log | tail -3
python scripts/bench_rpca.py 20 1 C4 > gpurun_out/rk_c4_64.json 2>/dev/null
UOT_RPCA_K=128 python scripts/bench_rpca.py 20 1 C4 > gpurun_out/rk_c4_128.json 2>/dev/null
for f in rk_c4_64 rk_c4_128; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); r=d['report']; print('$f', d['us_per_iter'], d['stage_us_per_iter'], r['objective'], r['svt_min_ritz'], r['nuclear'])"; done
