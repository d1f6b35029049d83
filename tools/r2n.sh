set -u
O=gpurun_out/r2n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hardening.py -q -x -s -k final > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/c5_combine.py fast > $O/c5_combine.log 2>&1; echo "c5comb rc=$?"
SGWG_LIB=paper_2007_10196_b200/libsgwg_f3.so timeout 600 python tools/c5_combine.py fast > $O/c5_combine_f3.log 2>&1; echo "c5comb rc=$?"
SGWG_LIB=paper_2007_10196_b200/libsgwg_f4.so timeout 600 python tools/c5_combine.py fast > $O/c5_combine_f4.log 2>&1; echo "c5comb rc=$?"
