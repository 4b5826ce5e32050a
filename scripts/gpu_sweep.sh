# Bench variants (env settings) on one config, one line each: bash scripts/gpu_sweep.sh CONFIG "ENV=.." ...
mkdir -p gpurun_out
cfg=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  env $e python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e ${BENCH_EXTRA:-} > gpurun_out/sweep_$i.log 2>&1
  tail -1 gpurun_out/sweep_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$e', '%.4e'%d['value'], round(d['ms_per_step'],2), r['kernel'][:12], round(r['frac'],3), d['clocks']['sm_mhz'], json.dumps({k:(round(v['ms']/v['launches'],3),v['launches']) for k,v in r['kernels_in_step'].items()}))" || tail -3 gpurun_out/sweep_$i.log
done
# (BENCH_EXTRA: extra bench.py arguments, e.g. "--mode prox")
