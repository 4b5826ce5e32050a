# chain prox (one-pass k_iter<PROX>): segment heights vs wave quantisation
for H in 8 16 32; do UOT_SEG_H=$H timeout 300 python bench.py --config C3 --mode prox --steps 2 --warmup 2 --no-e2e --no-cpu --iters 200 > gpurun_out/pxh_C3_$H.json 2>/dev/null; done
for H in 32 64 128; do UOT_SEG_H=$H timeout 300 python bench.py --mode prox --steps 2 --warmup 2 --no-e2e --no-cpu --iters 60 > gpurun_out/pxh_C4_$H.json 2>/dev/null; done
