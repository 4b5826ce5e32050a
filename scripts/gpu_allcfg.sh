# Full GPU test suite + bench on every config (fixed marginals), one line per config.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/all_tests.log 2>&1; tail -2 gpurun_out/all_tests.log
for c in ${CONFIGS:-C1 C2 C3 C4 C5}; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], d['ms_per_step'], r['kernel'][:14], round(r['frac'],3), json.dumps({k:(round(v['ms'],1),v['launches']) for k,v in r['kernels_in_step'].items()}))" || tail -3 gpurun_out/bench_$c.err
done
