# chain-prox one-pass kernel: register cap A/B (min blocks 4 = default vs 3) on C4
timeout 600 python bench.py --mode prox --steps 2 --warmup 2 --no-e2e --no-cpu --iters 100 > gpurun_out/prox_mb4.json 2>/dev/null
UOT_NVCC_EXTRA=-DUOT_PROX_MIN_BLOCKS=3 python paper_1909_00149_b200/build.py --force > /dev/null 2>&1
timeout 600 python bench.py --mode prox --steps 2 --warmup 2 --no-e2e --no-cpu --iters 100 > gpurun_out/prox_mb3.json 2>/dev/null
for v in 2 1; do UOT_VEC=$v timeout 600 python bench.py --mode prox --steps 2 --warmup 2 --no-e2e --no-cpu --iters 100 > gpurun_out/prox_mb3_v$v.json 2>/dev/null; done
