mkdir -p gpurun_out
run() { # label env... -- args
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu $BARGS 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$label', '%.3e'%d['value'], '%.0f'%r['achieved'], '%.3f'%r['frac'], '%.3f ms/it'%r['avg_launch_ms'])"
}
BARGS="--iters 100"
for V in 4 2; do run "C4 fixed V=$V" UOT_VEC=$V; done
BARGS="--iters 100 --mode prox"
for V in 4 2; do run "C4 prox V=$V" UOT_VEC=$V; done
for H in 32 64 128; do run "C4 prox V=2 H=$H" UOT_VEC=2 UOT_SEG_H=$H; done
BARGS="--config C3 --iters 300"
for V in 1 2 4; do for H in 4 8 16 32; do run "C3 fixed V=$V H=$H" UOT_VEC=$V UOT_SEG_H=$H; done; done
BARGS="--config C2 --iters 300"
for V in 1 2 4; do for H in 4 8 16; do run "C2 fixed V=$V H=$H" UOT_VEC=$V UOT_SEG_H=$H; done; done
BARGS="--config C1 --iters 300"
run "C1 fixed default"
BARGS="--config C5 --iters 60"
for V in 4 2; do run "C5 fixed V=$V" UOT_VEC=$V; done
