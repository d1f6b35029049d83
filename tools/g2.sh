set -u
O=gpurun_out/r4e; mkdir -p $O
echo "== gs 3"; timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof_3.json 2>&1; grep -A8 '"name"' $O/kprof_3.json | grep "avg_us"
for g in 2 4 5; do
echo "== gs $g"; SGWG_LIB=$PWD/tracelib/libsgwg_gs$g.so timeout 120 python tools/profile_c5.py C5 0.02 > $O/kprof_$g.json 2>&1; grep -A8 '"name"' $O/kprof_$g.json | grep "avg_us"
done
