mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python -m pytest tests/test_gpu_k1u.py -x -q -p no:cacheprovider > gpurun_out/a_k1u.log 2>&1; echo "k1u rc=$?"; tail -15 gpurun_out/a_k1u.log
