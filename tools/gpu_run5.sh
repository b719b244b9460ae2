timeout 600 python -m pytest tests/test_gpu_k1u.py -x -q -p no:cacheprovider > gpurun_out/g_k1u.log 2>&1; echo "k1u rc=$?"; tail -3 gpurun_out/g_k1u.log
bash tools/ab_k1.sh k1p0 k1p1
