# C2 (one 512^2 pair, 2000 iterations): the register wavefront with short segments vs the
# persistent SMEM-tile passes (default)
set -u
B="python bench.py --config C2 --no-cpu --no-e2e --steps 3 --warmup 3"
run() { echo "$1"; env $1 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernels_in_step'])"; }
run "UOT_DEBUG=0"
for h in 16 24 32 48 64 128; do run "UOT_WAVE=1 UOT_TPERSIST=0 UOT_WAVE_H=$h"; done
run "UOT_WAVE=1 UOT_TPERSIST=0 UOT_WAVE_H=32 UOT_WAVE_V=2"
run "UOT_WAVE=1 UOT_TPERSIST=0 UOT_WAVE_H=16 UOT_WAVE_V=2"
