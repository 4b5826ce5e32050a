# C3: wavefront segment heights that fit the warps in whole waves (forced wavefront)
for H in 16 32 37 43 52 64; do
  UOT_WAVE=1 UOT_WAVE_H=$H timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3w_H$H.json 2>/dev/null
done
