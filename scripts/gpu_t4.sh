# A/B of the temporally blocked variants on the default bench workload (C4).
# Usage: bash scripts/gpu_t4.sh ["ENV=.. ENV=.." ...]   (default: the variants below)
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "temporal or path or fixed" > gpurun_out/t4_tests.log 2>&1
tail -3 gpurun_out/t4_tests.log
if [ $# -eq 0 ]; then
  set -- "UOT_T4=0" "UOT_T4=1 UOT_T4_TH=32" "UOT_T4=1 UOT_T4_TH=36" "UOT_T4=1 UOT_T4_TH=40"
fi
for e in "$@"; do
  echo "== $e"
  env $e python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/t4_bench.log 2>&1
  tail -1 gpurun_out/t4_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%.3e'%d['value'], d['ms_per_step'], r['kernel'], r['frac'], r['avg_launch_ms'], json.dumps(r['kernels_in_step']))" || tail -5 gpurun_out/t4_bench.log
done
