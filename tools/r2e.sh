set -u
O=gpurun_out/r2e; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for mk in 1; do
  SGWG_P4_MASKED=$mk timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_m$mk.json 2>&1; echo "m $mk rc=$?"
  SGWG_P4_MASKED=$mk SGWG_P4_DBG=2 timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof_m${mk}_d2.json 2>&1; echo "m $mk rc=$?"
done
