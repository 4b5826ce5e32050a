# round 2: the whole -m gpu suite + smoke
python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/all_gpu.log 2>&1; echo EXIT $? >> gpurun_out/all_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT $? >> gpurun_out/smoke.log
