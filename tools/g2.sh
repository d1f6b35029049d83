set -u
O=gpurun_out/r4f; mkdir -p $O
timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof.json 2>&1; echo "rc=$?"; grep -A8 '"name"' $O/kprof.json | grep "name\|avg_us"
timeout 900 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py tests/test_gpu_fast.py -x -q -m gpu > $O/pytest_vp.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_vp.log
timeout 600 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -m gpu > $O/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_full.log
