timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_variants_gpu.py -q -x -m gpu > gpurun_out/quick.log 2>&1; echo EXIT $? >> gpurun_out/quick.log
for c in C3 C4; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bq_$c.json 2>/dev/null; done
