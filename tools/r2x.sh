set -u
O=gpurun_out/r2x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_fullsize_parity.py -k "final or c5_reduced or overflow" -q -x -s > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/c5_combine.py fast > $O/c5_combine.log 2>&1; echo "c5comb rc=$?"
SGWG_FINAL_NOSMEM=1 timeout 600 python tools/c5_combine.py fast > $O/c5_combine_nosmem.log 2>&1; echo "c5comb rc=$?"
