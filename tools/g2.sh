set -u
O=gpurun_out/r3k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py -x -q -m gpu > $O/pytest_vp.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_vp.log
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -m gpu -k "c5" > $O/pytest_c5.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_c5.log
python tools/profile_c5.py C5 0.02 > $O/kprof.json 2>&1; grep -A8 '"name"' $O/kprof.json | grep "name\|avg_us"
python tools/profile_evolve.py --config C5 --tfinal 2.0 > $O/plain2.log 2>&1; cat $O/plain2.log
