# chain prox (C4, rho = 10): k_wave_prox cluster size / segment height sweep
set -u
B="python bench.py --mode prox --no-cpu --no-e2e --steps 2 --warmup 3"
for cl in 2 4 8; do
  UOT_DEBUG=1 UOT_PROX_CL=$cl $B > gpurun_out/ps_cl$cl.json 2> gpurun_out/ps_cl$cl.err
done
for h in 128 256 1024; do
  UOT_PROX_WAVE_H=$h $B > gpurun_out/ps_h$h.json 2> gpurun_out/ps_h$h.err
done
for f in gpurun_out/ps_*.json; do echo $f; grep -h "plan" ${f%.json}.err | head -1; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"; done
