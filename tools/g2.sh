set -u
O=gpurun_out/r4h; mkdir -p $O
echo "== base (13-value window)"; timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof_b.json 2>&1; grep -A8 '"name"' $O/kprof_b.json | grep "avg_us"
for v in h1 h1g5; do
echo "== $v"; SGWG_LIB=$PWD/tracelib/libsgwg_$v.so timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof_$v.json 2>&1; grep -A8 '"name"' $O/kprof_$v.json | grep "avg_us"
done
SGWG_LIB=$PWD/tracelib/libsgwg_h1.so timeout 600 python -m pytest tests/test_gpu_vp.py -x -q -m gpu > $O/pytest_vp.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_vp.log
