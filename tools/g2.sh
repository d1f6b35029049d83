set -u
O=gpurun_out/r4g; mkdir -p $O
echo "== batch 5"; timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof_5.json 2>&1; grep -A8 '"name"' $O/kprof_5.json | grep "avg_us" | head -1
for b in 3 9; do
echo "== batch $b"; SGWG_LIB=$PWD/tracelib/libsgwg_eb$b.so timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof_$b.json 2>&1; grep -A8 '"name"' $O/kprof_$b.json | grep "avg_us" | head -1
done
timeout 600 python -m pytest tests/test_gpu_vp.py -x -q -m gpu > $O/pytest_vp.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_vp.log
