# round 2, second measurement pass (k_wave_pk, k_wave_prox): default bench line (C4), the other
# configs, chain prox, the ncu launch lists of the default and chain-prox commands and --set full
# captures of k_wave_pk<5> (C4 fixed) and k_wave_prox<3> (C4 chain prox), summarised on the box
# (raw + source CSV; the binary reports stay there)
set -u
python bench.py > gpurun_out/r02b_bench_C4.json 2> gpurun_out/r02b_bench_C4.err; echo "EXIT $?" >> gpurun_out/r02b_bench_C4.err
for c in C5 C3 C2 C1; do
  python bench.py --config $c --no-cpu > gpurun_out/r02b_bench_$c.json 2> gpurun_out/r02b_bench_$c.err; echo "EXIT $?" >> gpurun_out/r02b_bench_$c.err
done
python bench.py --mode prox --no-cpu > gpurun_out/r02b_bench_C4_prox.json 2> gpurun_out/r02b_bench_C4_prox.err
python bench.py --config C3 --mode prox --no-cpu > gpurun_out/r02b_bench_C3_prox.json 2> gpurun_out/r02b_bench_C3_prox.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/r02b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_C4.csv $CMD > gpurun_out/r02b_ncu_launch.log 2>&1
PCMD="python bench.py --mode prox --steps 1 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_C4_prox.csv $PCMD > gpurun_out/r02b_ncu_launch_prox.log 2>&1
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:k_wave_pk -s 40 -c 2 -o /tmp/ncu/pk5 $CMD > gpurun_out/r02b_ncu_full.log 2>&1
echo "EXIT $?" >> gpurun_out/r02b_ncu_full.log
ncu -i /tmp/ncu/pk5.ncu-rep --page raw --csv > gpurun_out/r02b_k_wave_pk5_C4.raw.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_wave_prox -s 20 -c 1 -o /tmp/ncu/wp $PCMD > gpurun_out/r02b_ncu_full_prox.log 2>&1
echo "EXIT $?" >> gpurun_out/r02b_ncu_full_prox.log
ncu -i /tmp/ncu/wp.ncu-rep --page raw --csv > gpurun_out/r02b_k_wave_prox_C4.raw.csv 2>&1
ncu -i /tmp/ncu/wp.ncu-rep --page source --csv --print-source sass > gpurun_out/r02b_k_wave_prox_C4.src.csv 2>&1
gzip -f gpurun_out/*.csv
du -sh gpurun_out
for f in gpurun_out/r02b_bench_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], (d.get('e2e') or {}).get('value'), d['clocks'])"; done
