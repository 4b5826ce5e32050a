# chain prox A/B: M_y of the previous row in registers (uy0) or shared memory (uy1); needs
# libuot_uy0.so / libuot_uy1.so built with -DUOT_PROX_UY=0 / 1 at the repo root
set -u
B="python bench.py --mode prox --no-cpu --no-e2e --steps 3 --warmup 3"
for v in uy0 uy1 uy0 uy1; do
  cp libuot_$v.so paper_1909_00149_b200/libuot_b200.so
  for ps in 2 3; do
    echo "$v pass$ps $(UOT_PROX_PASS=$ps $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])")"
  done
done
