set -u
O=gpurun_out/r2l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_fast.py tests/test_gpu_diag.py tests/test_gpu_vp.py tests/test_gpu_convergence.py -q -x -s > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/c5_combine.py fast > $O/c5_combine.log 2>&1; echo "c5comb rc=$?"
SGWG_UPSAMPLE_GENERIC=1 timeout 600 python tools/c5_combine.py fast > $O/c5_combine_gen.log 2>&1; echo "c5comb rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_combine.csv python tools/c5_combine.py fast > $O/ncu_lc.log 2>&1; echo "ncu launches comb rc=$?"
