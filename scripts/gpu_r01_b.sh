mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_all.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_c4_fixed.log 2>&1; echo b1=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --mode prox > gpurun_out/b_c4_prox.log 2>&1; echo b2=$?
timeout 300 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu --mode prox > gpurun_out/b_c3_prox.log 2>&1; echo b3=$?
for f in b_c4_fixed b_c4_prox b_c3_prox; do tail -1 gpurun_out/$f.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$f', '%.3e'%d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['ms_per_step'], d['e2e']['value'] if d['e2e'] else None)"; done
