# ncu captures of the k_wave variants on C4 (20 iterations: S = 3 + 3 + 4 ... passes)
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-cpu --no-e2e --iters 20"
python bench.py $ARGS > gpurun_out/p.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_wave -s 6 -c 3 -o gpurun_out/kw -f python bench.py $ARGS > gpurun_out/kw_ncu.log 2>&1
tail -2 gpurun_out/kw_ncu.log
