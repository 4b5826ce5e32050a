# Algorithm 3 on the C3 video: exact Jacobi SVT vs the subspace partial SVD with small k
timeout 600 python scripts/bench_rpca.py 200 1 C3 > gpurun_out/rk_jacobi.json 2>/dev/null
for k in 8 16 32; do UOT_RPCA_SVT=1 UOT_RPCA_K=$k timeout 600 python scripts/bench_rpca.py 200 1 C3 > gpurun_out/rk_$k.json 2>/dev/null; done
