mkdir -p gpurun_out
set -x
timeout 600 python -m pytest tests -m gpu -q -k C4 > gpurun_out/gpu_c4.log 2>&1; echo c4=$?
for H in 16 32 64 128 256; do UOT_SEG_H=$H timeout 200 python bench.py --steps 2 --warmup 2 --iters 100 --no-e2e --no-cpu 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('H=$H', d['value'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'])"; done > gpurun_out/sweepH.log 2>&1
for C in C2 C3 C5; do timeout 400 python bench.py --config $C --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_$C.log 2>&1; echo $C=$?; done
timeout 400 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo l=$?
timeout 300 python bench.py --steps 1 --warmup 1 --iters 30 --no-e2e --no-cpu > gpurun_out/b30.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_fixed -s 20 -c 1 -o gpurun_out/prof_c4_r01 python bench.py --steps 1 --warmup 1 --iters 30 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo f=$?
