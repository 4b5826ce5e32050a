# C2: short-segment wavefront with shorter passes (latency per row step grows with S)
set -u
B="python bench.py --config C2 --no-cpu --no-e2e --steps 3 --warmup 3"
run() { echo "$1"; env $1 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernels_in_step'])"; }
for pc in "0.1,9,9,9" "9,0.1,9,9" "9,9,0.1,9"; do
  for v in 4 2; do run "UOT_WAVE=1 UOT_TPERSIST=0 UOT_WAVE_H=16 UOT_WAVE_V=$v UOT_PASS_COST=$pc"; done
done
