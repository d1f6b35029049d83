set -u
O=gpurun_out/r2f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for ps in 1 0; do
  SGWG_P4_PERSIST=$ps timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_p$ps.json 2>&1; echo "p $ps rc=$?"
done
SGWG_P4_VTARGET=2000 timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_p1_vt2000.json 2>&1; echo "vt rc=$?"
