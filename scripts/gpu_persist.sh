mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_prox_gpu.py -x -q -k "not C4 and not C5" > gpurun_out/persist_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/persist_tests.log
for C in C1 C2; do timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > gpurun_out/b_$C.log 2>&1; echo $C=$?; tail -1 gpurun_out/b_$C.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$C', '%.3e'%d['value'], '%.0f'%r['achieved'], '%.4f ms/it'%r['avg_launch_ms'], d['ms_per_step'], d['gpu_launches'])"; done
