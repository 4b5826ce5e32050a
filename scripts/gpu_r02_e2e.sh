# e2e pipelining: pair ranges on K streams (4 vs 8)
for K in 4 8; do
  timeout 600 python bench.py --no-cpu --e2e-chunks $K > gpurun_out/e2e_K$K.json 2>/dev/null
done
