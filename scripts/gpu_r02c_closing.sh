# round 2 closing run: the full GPU suite + smoke, then the default bench line
set -u
bash scripts/gpu_r02_alltests.sh
python bench.py > gpurun_out/r02c_bench_C4_final.json 2> gpurun_out/r02c_bench_C4_final.err
python -c "import json; d=json.loads(open('gpurun_out/r02c_bench_C4_final.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
