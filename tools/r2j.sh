set -u
O=gpurun_out/r2j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vp.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for ps in 1 0; do
  SGWG_P4_PERSIST=$ps timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_p$ps.json 2>&1; echo "p $ps rc=$?"
done
SGWG_LIB=paper_2007_10196_b200/libsgwg_trace.so timeout 300 python tools/trace_p4p.py > $O/trace.txt 2>&1
