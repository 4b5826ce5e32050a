# C3 fixed: pass length (UOT_PASS_COST forcing S = 3 / 4 / 5) x segment height
set -u
B="python bench.py --config C3 --no-cpu --no-e2e --steps 3 --warmup 3"
run() { echo "$1"; env $1 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernels_in_step'])"; }
run "UOT_PASS_COST=1.155,1.15,1.137,1.35"
run "UOT_PASS_COST=9,9,0.1,9"
run "UOT_PASS_COST=9,0.1,9,9"
run "UOT_PASS_COST=9,9,0.1,9 UOT_WAVE_H=32"
run "UOT_PASS_COST=9,9,0.1,9 UOT_WAVE_H=52"
run "UOT_WAVE_H=37"
run "UOT_WAVE_H=52"
run "UOT_WAVE_H=64"
