# ncu full capture of k_single on C1 (after a plain run of the same command)
CMD="python bench.py --config C1 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_single.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_single -s 3 -c 1 -o gpurun_out/single_c1 $CMD > gpurun_out/ncu_single.log 2>&1
echo EXIT $? >> gpurun_out/ncu_single.log
