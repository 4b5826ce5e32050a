# C3 chain prox on the one-pass k_iter<PROX>: lane width x segment rows
set -u
B="python bench.py --config C3 --mode prox --no-cpu --no-e2e --steps 2 --warmup 3"
run() { echo "$1"; env $1 UOT_DEBUG=0 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"; }
run "UOT_VEC=0"
for v in 4 2 1; do for h in 8 16 32 64; do run "UOT_VEC=$v UOT_SEG_H=$h"; done; done
