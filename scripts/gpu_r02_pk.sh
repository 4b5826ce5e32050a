# packed fp32x2 k_wave (k_wave_pk) vs scalar k_wave: parity subset + C4/C3/C5 bench A/B
set -u
python -m pytest tests/test_parity_gpu.py -x -q -k "wave_edge or random_pass or temporal_matches or C4_subset or C3_subset or C5 or checkpoint" > gpurun_out/pk_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/pk_tests.log
for pk in 1 0; do
  UOT_WAVE_PK=$pk python bench.py --no-cpu --no-e2e > gpurun_out/pk${pk}_C4.json 2> gpurun_out/pk${pk}_C4.err
  UOT_WAVE_PK=$pk python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/pk${pk}_C3.json 2> gpurun_out/pk${pk}_C3.err
done
UOT_WAVE_PK=1 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/pk1_C5.json 2> gpurun_out/pk1_C5.err
tail -3 gpurun_out/pk_tests.log; for f in gpurun_out/pk*_C*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done
