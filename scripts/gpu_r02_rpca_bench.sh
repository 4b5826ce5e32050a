# Algorithm 3 timings: C3 video (T = 64, exact Jacobi SVT) and C4 video (T = 256, partial SVD)
timeout 600 python scripts/bench_rpca.py 200 1 C3 > gpurun_out/r02_rpca_c3.json 2> gpurun_out/r02_rpca_c3.err
timeout 900 python scripts/bench_rpca.py 20 1 C4 > gpurun_out/r02_rpca_c4.json 2> gpurun_out/r02_rpca_c4.err
echo done
