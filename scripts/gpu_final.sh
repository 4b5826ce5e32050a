# Round-end measurement set: GPU tests, smoke, bench lines for every config (+ chain prox),
# ncu launch list of the default bench command and a full capture of the dominant kernel.
mkdir -p gpurun_out/final
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/tests.log 2>&1; tail -1 gpurun_out/final/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -3 gpurun_out/final/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/final/bench_C4.json 2> gpurun_out/final/bench_C4.err; echo C4=$?
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; echo $c=$?; done
for c in C3 C4; do timeout 900 python bench.py --config $c --mode prox --steps 2 --warmup 3 --no-cpu > gpurun_out/final/bench_${c}_prox.json 2> gpurun_out/final/bench_${c}_prox.err; echo ${c}prox=$?; done
timeout 900 python scripts/bench_fig1.py --out gpurun_out/final/fig1.md > gpurun_out/final/fig1.log 2>&1; echo fig1=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final/ncu_launch.log 2>&1; echo launches=$?
ARGS="--steps 1 --warmup 3 --no-cpu --no-e2e --iters 20"
timeout 300 python bench.py $ARGS > gpurun_out/final/b20.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 4 -c 2 -o gpurun_out/final/prof_k_wave5_C4 -f python bench.py $ARGS > gpurun_out/final/ncu_full.log 2>&1; echo full=$?
