set -u
O=gpurun_out/r2v; mkdir -p $O
SGWG_P4_XPERSIST=1 timeout 900 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for xp in 0 1; do
  SGWG_P4_XPERSIST=$xp timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_xp$xp.json 2>&1; echo "xp $xp rc=$?"
done
SGWG_P4_XPERSIST=1 SGWG_LIB=paper_2007_10196_b200/libsgwg_trace.so timeout 300 python tools/trace_x4p.py > $O/trace.txt 2>&1
