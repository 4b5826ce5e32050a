# round 2, third measurement pass (final kernels): bench lines of every config and of chain prox,
# ncu launch lists of the default and chain-prox commands, a --set full capture of k_wave_pk<5>
# (raw + source pages exported on the box), then the full GPU suite + smoke
set -u
python bench.py > gpurun_out/r02c_bench_C4.json 2> gpurun_out/r02c_bench_C4.err; echo "EXIT $?" >> gpurun_out/r02c_bench_C4.err
for c in C5 C3 C2 C1; do
  python bench.py --config $c --no-cpu > gpurun_out/r02c_bench_$c.json 2> gpurun_out/r02c_bench_$c.err; echo "EXIT $?" >> gpurun_out/r02c_bench_$c.err
done
python bench.py --mode prox --no-cpu > gpurun_out/r02c_bench_C4_prox.json 2> gpurun_out/r02c_bench_C4_prox.err
python bench.py --config C3 --mode prox --no-cpu > gpurun_out/r02c_bench_C3_prox.json 2> gpurun_out/r02c_bench_C3_prox.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02c_bench_ref.json 2> gpurun_out/r02c_bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/r02c_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_C4.csv $CMD > gpurun_out/r02c_ncu_launch.log 2>&1
PCMD="python bench.py --mode prox --steps 1 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_C4_prox.csv $PCMD > gpurun_out/r02c_ncu_launch_prox.log 2>&1
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:k_wave_pk -s 40 -c 2 -o /tmp/ncu/pk5 $CMD > gpurun_out/r02c_ncu_full.log 2>&1
echo "EXIT $?" >> gpurun_out/r02c_ncu_full.log
ncu -i /tmp/ncu/pk5.ncu-rep --page raw --csv > gpurun_out/r02c_k_wave_pk5_C4.raw.csv 2>&1
ncu -i /tmp/ncu/pk5.ncu-rep --page source --csv --print-source sass > gpurun_out/r02c_k_wave_pk5_C4.src.csv 2>&1
python scripts/bench_rpca.py 200 > gpurun_out/r02c_rpca_c3.json 2> gpurun_out/r02c_rpca_c3.err
gzip -f gpurun_out/r02c_*.csv
bash scripts/gpu_r02_alltests.sh
for f in gpurun_out/r02c_bench_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; print(d['value'], d.get('ms_per_step'), r.get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks'))"; done
