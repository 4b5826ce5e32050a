set -u
B="python bench.py --mode prox --no-cpu --no-e2e --steps 3 --warmup 3"
timeout 900 python -m pytest -x -q tests/test_prox_wave_gpu.py > gpurun_out/r4_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/r4_tests.log; tail -2 gpurun_out/r4_tests.log
$B > gpurun_out/r4_a.json 2>/dev/null
UOT_PROX_PASS=3 $B > gpurun_out/r4_p3.json 2>/dev/null
cp paper_1909_00149_b200/libuot_b200.so /tmp/ring4.so
cp libuot_ring3.so paper_1909_00149_b200/libuot_b200.so
$B > gpurun_out/r3_a.json 2>/dev/null
UOT_PROX_PASS=3 $B > gpurun_out/r3_p3.json 2>/dev/null
cp /tmp/ring4.so paper_1909_00149_b200/libuot_b200.so
$B > gpurun_out/r4_b.json 2>/dev/null
for f in r4_a r4_p3 r3_a r3_p3 r4_b; do echo $f; python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
