set -u
O=gpurun_out/g6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_vp.py tests/test_gpu_fast.py -q -x -s > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 300 python tools/profile_c5.py C5 0.02 > $O/prof.json 2> $O/prof.err; echo "prof rc=$?"
timeout 600 python tools/c5_combine.py fast > $O/c5_combine.log 2>&1; echo "c5comb rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"xpass4d|vpass4d" -s 6 -c 2 -o $O/p4 python tools/profile_c5.py C5 0.01 > $O/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_comb.csv python tools/c5_combine.py fast > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?"
