# UOT-DF wavefront segment heights (Fig. 1 sizes): model vs round 1's rule
timeout 600 python scripts/bench_fig1.py --sizes 1024,2048,4096 --out gpurun_out/fig1_model.md > gpurun_out/fig1_model.log 2>&1
UOT_WAVE_H=64 timeout 600 python scripts/bench_fig1.py --sizes 4096 --out gpurun_out/fig1_h64.md > gpurun_out/fig1_h64.log 2>&1
timeout 900 python -m pytest tests/test_df_gpu.py -q -x -m gpu > gpurun_out/df.log 2>&1; echo EXIT $? >> gpurun_out/df.log
