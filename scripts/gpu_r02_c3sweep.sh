# C3 geometry sweep: wavefront segment rows and pass lengths
for H in 16 32 64 128; do
  UOT_WAVE_H=$H python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_H$H.json 2>/dev/null
done
for pc in "1.155,1.15,1.137,9" "1.155,1.15,9,9"; do
  UOT_PASS_COST=$pc python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > "gpurun_out/c3_pc_$pc.json" 2>/dev/null
done
