# round 2 measurement + profiles: default bench line (C4), the other configs, chain prox,
# the ncu launch list of the default command and one --set full capture of k_wave<5>
set -u
python bench.py > gpurun_out/r02_bench_C4.json 2> gpurun_out/r02_bench_C4.err; echo "EXIT $?" >> gpurun_out/r02_bench_C4.err
for c in C5 C3 C2 C1; do
  python bench.py --config $c --no-cpu > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "EXIT $?" >> gpurun_out/r02_bench_$c.err
done
python bench.py --mode prox --no-cpu > gpurun_out/r02_bench_C4_prox.json 2> gpurun_out/r02_bench_C4_prox.err; echo "EXIT $?" >> gpurun_out/r02_bench_C4_prox.err
python bench.py --config C3 --mode prox --no-cpu > gpurun_out/r02_bench_C3_prox.json 2> gpurun_out/r02_bench_C3_prox.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/r02_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_C4.csv $CMD > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_wave -s 40 -c 2 -o gpurun_out/r02_k_wave5_C4 $CMD > gpurun_out/r02_ncu_full.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_ncu_full.log
