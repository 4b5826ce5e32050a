# k_single (C1): bench with 8 and 4 pixels per thread, then an ncu --set full capture with the
# source page (stall reasons per SASS line) exported on the box
set -u
B="python bench.py --config C1 --no-cpu --steps 3 --warmup 3"
$B > gpurun_out/s_C1_v8.json 2> gpurun_out/s_C1_v8.err
UOT_SINGLE_V=4 $B > gpurun_out/s_C1_v4.json 2> gpurun_out/s_C1_v4.err
for f in gpurun_out/s_C1_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks'])"; done
CMD="python bench.py --config C1 --steps 2 --warmup 3 --no-e2e --no-cpu"
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:k_single -s 3 -c 1 -o /tmp/ncu/single $CMD > gpurun_out/s_ncu.log 2>&1
echo EXIT $? >> gpurun_out/s_ncu.log
ncu -i /tmp/ncu/single.ncu-rep --page raw --csv > gpurun_out/s_single_raw.csv 2>&1
ncu -i /tmp/ncu/single.ncu-rep --page source --csv --print-source sass > gpurun_out/s_single_src.csv 2>&1
ncu -i /tmp/ncu/single.ncu-rep --page details --csv > gpurun_out/s_single_details.csv 2>&1
gzip -f gpurun_out/s_single_*.csv
