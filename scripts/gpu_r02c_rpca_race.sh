# RPCA T > 128 multi-wave apply: sharded-vs-unsharded bitwise on 128 x 128 frames with the fixed
# library, then with the library built from the previous sources (libuot_old.so at the repo root,
# D written inside the apply)
set -u
T="tests/test_rpca_big_gpu.py -k sharded_bitwise_frames"
timeout 900 python -m pytest -q $T > gpurun_out/race_new.log 2>&1; echo "EXIT $?" >> gpurun_out/race_new.log
grep -E "AssertionError|passed|failed" gpurun_out/race_new.log | tail -3
cp paper_1909_00149_b200/libuot_b200.so /tmp/new.so
cp libuot_old.so paper_1909_00149_b200/libuot_b200.so
timeout 900 python -m pytest -q $T > gpurun_out/race_old.log 2>&1; echo "EXIT $?" >> gpurun_out/race_old.log
grep -E "AssertionError|passed|failed" gpurun_out/race_old.log | tail -3
cp /tmp/new.so paper_1909_00149_b200/libuot_b200.so
