# ncu --set full capture of k_wave_prox<2> (C4 chain prox, passes of 2), raw + source pages exported
set -u
PCMD="python bench.py --mode prox --steps 1 --warmup 3 --no-e2e --no-cpu"
$PCMD > gpurun_out/p2_plain.log 2>&1
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:k_wave_prox -s 20 -c 1 -o /tmp/ncu/wp2 $PCMD > gpurun_out/p2_ncu.log 2>&1
echo "EXIT $?" >> gpurun_out/p2_ncu.log
ncu -i /tmp/ncu/wp2.ncu-rep --page raw --csv > gpurun_out/p2_raw.csv 2>&1
ncu -i /tmp/ncu/wp2.ncu-rep --page source --csv --print-source sass > gpurun_out/p2_src.csv 2>&1
gzip -f gpurun_out/p2_*.csv
tail -2 gpurun_out/p2_ncu.log
