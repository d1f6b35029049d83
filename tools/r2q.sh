set -u
O=gpurun_out/r2q; mkdir -p $O
export SGWG_LIB=paper_2007_10196_b200/libsgwg_check.so
timeout 600 python tools/sanitize_cases.py > $O/cases.log 2>&1; echo "cases rc=$?"
SGWG_P4_PERSIST=0 timeout 600 python tools/sanitize_cases.py C5 > $O/cases_np.log 2>&1; echo "cases np rc=$?"
timeout 600 python tools/profile_c5.py C5 0.01 > $O/c5prof.log 2>&1; echo "c5 full-size evolve rc=$?"
timeout 900 python tools/c5_combine.py fast > $O/c5comb.log 2>&1; echo "c5 full combine rc=$?"
timeout 1200 python -m pytest tests/test_gpu_vp.py tests/test_gpu_hardening.py tests/test_gpu_fast.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
