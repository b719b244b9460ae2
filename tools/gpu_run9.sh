timeout 900 python -m pytest tests/test_gpu_kron.py -x -q -p no:cacheprovider > gpurun_out/l_kron.log 2>&1; echo "kron rc=$?"; tail -30 gpurun_out/l_kron.log | head -60
