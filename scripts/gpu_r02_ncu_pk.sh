# ncu full capture of k_wave_pk<5> and scalar k_wave<5> on C4 (after a plain run of the same command)
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_pk.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_wave -s 40 -c 1 -o gpurun_out/r02_k_wave_pk5_C4 $CMD > gpurun_out/ncu_pk.log 2>&1
echo EXIT $? >> gpurun_out/ncu_pk.log
UOT_WAVE_PK=0 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 40 -c 1 -o gpurun_out/r02_k_wave5_C4_scalar $CMD > gpurun_out/ncu_sc.log 2>&1
echo EXIT $? >> gpurun_out/ncu_sc.log
