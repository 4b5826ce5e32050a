mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_prox_gpu.py -x -q -k "not C4 and not C5" > gpurun_out/persist_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/persist_tests.log
b() { local label=$1; shift; env "$@" timeout 300 python bench.py $BARGS --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$label', '%.3e'%d['value'], '%.0f'%r['achieved'], '%.4f ms/it'%r['avg_launch_ms'], d['ms_per_step'])"; }
BARGS="--config C1"
b "C1 auto(1 tile)"; b "C1 32x16" UOT_TILE=32x16; b "C1 32x32" UOT_TILE=32x32; b "C1 16x16" UOT_TILE=16x16; b "C1 stream" UOT_PERSIST=0
BARGS="--config C2"
b "C2 auto(64x32)"; b "C2 32x32" UOT_TILE=32x32; b "C2 64x64" UOT_TILE=64x64; b "C2 128x64" UOT_TILE=128x64; b "C2 stream" UOT_PERSIST=0
python bench.py --config C2 --iters 200 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/c2p.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o gpurun_out/prof_c2_persist python bench.py --config C2 --iters 200 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
