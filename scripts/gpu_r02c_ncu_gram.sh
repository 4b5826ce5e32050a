# ncu --set full of the pipelined Gram (C4 video), raw + source pages exported on the box
set -u
CMD="python scripts/bench_rpca.py 2 1 C4"
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:k_rp_gram_pipe -s 1 -c 1 -o /tmp/ncu/gram $CMD > gpurun_out/gr_ncu.log 2>&1
echo "EXIT $?" >> gpurun_out/gr_ncu.log
ncu -i /tmp/ncu/gram.ncu-rep --page raw --csv > gpurun_out/gr_raw.csv 2>&1
ncu -i /tmp/ncu/gram.ncu-rep --page source --csv --print-source sass > gpurun_out/gr_src.csv 2>&1
gzip -f gpurun_out/gr_*.csv
tail -2 gpurun_out/gr_ncu.log
