# Bench line + ncu launch list of the same command + full ncu capture of the k_wave passes (C4).
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err; echo b=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_wave.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo l=$?
ARGS="--steps 1 --warmup 3 --no-cpu --no-e2e --iters 20"
timeout 300 python bench.py $ARGS > gpurun_out/b20.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 6 -c 3 -o gpurun_out/prof_wave_C4 -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo f=$?
